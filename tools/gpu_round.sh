#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list + full capture.
# usage: tools/gpu_round.sh <tag> [parts...]   parts: tests smoke bench launches full
set -u
TAG=${1:-r01}; shift || true
PARTS=${@:-tests smoke bench launches full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
for p in $PARTS; do
  case $p in
    tests)  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cp gpurun_out/clocks_rank0.csv $OUT/ 2>/dev/null ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
          --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" ;;
    full)   timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_material -s 3 -c 1 \
          -o $OUT/material python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 262144 > $OUT/full.log 2>&1; echo "full rc=$?" ;;
  esac
done
