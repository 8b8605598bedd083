set -u
O=gpurun_out/r21; mkdir -p $O
L=paper_2006_04391_b200/libautomat.so
ncu --set full --clock-control none --import-source on -k regex:k_material -s 3 -c 1 -o $O/k1_newton python tools/k1_variants.py --one $L 262144 > $O/ncu1.log 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:k_tangent -s 3 -c 1 -o $O/k1_tangent python tools/k1_variants.py --one $L 262144 > $O/ncu2.log 2>&1; echo ncu2 $?
ncu --set full --clock-control none --import-source on -k regex:"k_fourier|k_material" -s 2 -c 4 -o $O/basic256 python tools/basic_profile.py 256 3 > $O/ncu3.log 2>&1; echo ncu3 $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --basic 64 --path 0 > $O/launches_bench.log 2>&1; echo launches $?
python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
