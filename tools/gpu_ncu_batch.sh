# ncu of the batch kernel on the current build: launch list of the default bench
# (1 step) and one --set full capture of k_track_batch (prof_batch.py dd 296 12:
# launch 3 = the measured launch after the workspace warm-up); only summaries return
O=gpurun_out/r02ncu; mkdir -p $O; R=/tmp/ncu_batch
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/launches_batch32_dd.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/launches.log 2>&1
echo "launch list rc=$?"
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:k_track_batch --launch-skip 2 -c 1 -o $R \
  python tools/prof_batch.py dd 296 12 > $O/ncu_full.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py $R.ncu-rep batch32_dd > $O/ncu_full_batch32_dd.json
ncu -i $R.ncu-rep --page details --csv > $O/ncu_details_batch32_dd.csv 2>/dev/null
head -c 1500 $O/ncu_full_batch32_dd.json
