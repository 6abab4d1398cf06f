mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track -c 1 -o gpurun_out/prof_${1}_${2} python tools/one_path.py $1 $2 > gpurun_out/ncu_${1}_${2}.log 2>&1
tail -2 gpurun_out/ncu_${1}_${2}.log
