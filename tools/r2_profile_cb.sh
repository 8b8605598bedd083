OUT=gpurun_out/r2cb
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $OUT/launches_basic256_cb.csv python tools/basic_profile.py 256 6 > $OUT/launches.log 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fourier" -s 2 -c 1 -o $OUT/fourier256_cb python tools/basic_profile.py 256 4 > $OUT/full.log 2>&1
echo "full rc=$?"
for r in $OUT/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; done
ls -la $OUT
