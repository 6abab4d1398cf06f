#!/bin/bash
# first measurement session: FP64 peak, benches, reference arm, ncu launch list + full capture
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt
timeout 120 python tools/measure_fp64_peak.py > gpurun_out/fp64.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_chandra_dd.json 2> gpurun_out/bench_chandra_dd.err
timeout 300 python bench.py --steps 10 --warmup 3 --prec d --no-cpu-baseline > gpurun_out/bench_chandra_d.json 2> gpurun_out/bench_chandra_d.err
timeout 600 python bench.py --steps 5 --warmup 3 --prec qd --no-cpu-baseline > gpurun_out/bench_chandra_qd.json 2> gpurun_out/bench_chandra_qd.err
timeout 300 python bench.py --steps 10 --warmup 3 --workload cyclic16 --no-cpu-baseline > gpurun_out/bench_cyclic16_dd.json 2> gpurun_out/bench_cyclic16_dd.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
lscpu > gpurun_out/lscpu.txt; nproc > gpurun_out/nproc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_chandra_dd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_track_grid -c 1 -o gpurun_out/prof_chandra_dd python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
