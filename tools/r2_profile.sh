#!/bin/bash
# Round-2 ncu evidence (GPU box): launch lists (cold-cache, serialised
# per-launch times) and --set full captures of the dominant kernels.
# usage: tools/r2_profile.sh <out dir under gpurun_out>
set -u
OUT=gpurun_out/${1:-r2prof}
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --basic 0 --path 0 --big 0 --no-strategies"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_config2.csv $B > $OUT/launches_config2.log 2>&1
echo "launches config2 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_material|k_tangent" -s 6 -c 2 \
    -o $OUT/k1_config2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --basic 0 --path 0 --big 0 --no-strategies > $OUT/full_config2.log 2>&1
echo "full config2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_basic256.csv \
    python tools/basic_variants.py --one paper_2006_04391_b200/libautomat.so 256 6 > $OUT/launches_basic256.log 2>&1
echo "launches basic rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_material|k_fourier" -s 6 -c 3 \
    -o $OUT/basic256 python tools/basic_variants.py --one paper_2006_04391_b200/libautomat.so 256 4 > $OUT/full_basic256.log 2>&1
echo "full basic rc=$?"
for r in $OUT/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; done
ls -la $OUT
