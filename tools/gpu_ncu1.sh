mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track -c 1 -o gpurun_out/prof_chandra_d python tools/one_path.py chandra64 d > gpurun_out/ncu_d.log 2>&1
tail -3 gpurun_out/ncu_d.log
