set -u
O=gpurun_out/r08; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_basic256.csv python tools/basic_profile.py 256 3 > $O/launches_basic.log 2>&1; echo launches $?
ncu --set full --clock-control none --import-source on -k regex:"k_fourier|k_material" -s 2 -c 4 -o $O/basic256 python tools/basic_profile.py 256 3 > $O/full_basic.log 2>&1; echo full $?
