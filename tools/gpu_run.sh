# final-build evidence for the headline kernel: ncu launch list of the default bench + one full capture
O=gpurun_out/r02ncufinal; mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file $O/launches_batch32_dd.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
r=/tmp/bfinal
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:k_track_batch --launch-skip 2 -c 1 -o $r python tools/prof_batch.py dd 296 12 > $O/ncu.log 2>&1
python tools/ncu_summary.py $r.ncu-rep batch32_dd > $O/ncu_full_batch32_dd.json
ncu -i $r.ncu-rep --page details --csv > $O/ncu_details_batch32_dd.csv 2>/dev/null
ncu -i $r.ncu-rep --page raw --csv > $O/ncu_raw_batch32_dd.csv 2>/dev/null
ncu -i $r.ncu-rep --page source --csv > $O/ncu_src_batch32_dd.csv 2>/dev/null; gzip -f $O/ncu_src_batch32_dd.csv
ls -la $O
