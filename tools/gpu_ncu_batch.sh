mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track_batch -c 1 -o gpurun_out/prof_batch_dd python tools/prof_batch.py dd 296 > gpurun_out/ncu_batch.log 2>&1
tail -2 gpurun_out/ncu_batch.log
