#!/bin/bash
# Build libautomat variants (kernel tuning experiments) into tools/variants/.
# usage: tools/build_variants.sh name "extra nvcc flags" [name flags ...]
set -e
cd "$(dirname "$0")/../paper_2006_04391_b200/csrc"
ARCH="-gencode arch=compute_100a,code=sm_100a"
NCCL_HOME=${NCCL_HOME:-/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl}
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=../../tools/variants/$name; mkdir -p $d
  for f in api material probe solver fft_cb k1_ms k1_ms_semi k1_adapt_ms k1_adapt_ms_semi k1_misc; do
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -I$NCCL_HOME/include $flags -c $f.cu -o $d/$f.o 2> $d/$f.ptxas.log &
  done
  wait
  nvcc $ARCH -shared -o $d/libautomat.so $d/*.o -lcudart -lcufft -ldl -L$NCCL_HOME/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL_HOME/lib
  echo "$name: $(grep -A2 'k_materialINS_15MichelSuquetLawELi0ELb0' $d/k1_ms.ptxas.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
