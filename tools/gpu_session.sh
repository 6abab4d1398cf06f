#!/bin/bash
# measurement session: default bench (+CPU baseline), reference arm, other configs,
# ncu launch list of the default command and one full ncu capture of the tracker kernel
set -x
mkdir -p gpurun_out/s
O=gpurun_out/s
nvidia-smi > $O/nvidia_smi.txt
lscpu > $O/lscpu.txt; nproc > $O/nproc.txt
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python bench.py --prec d --no-cpu-baseline > $O/bench_chandra_d.json 2> $O/bench_chandra_d.err
timeout 600 python bench.py --prec qd --steps 3 --no-cpu-baseline > $O/bench_chandra_qd.json 2> $O/bench_chandra_qd.err
timeout 300 python bench.py --workload cyclic16 --no-cpu-baseline > $O/bench_cyclic16_dd.json 2> $O/bench_cyclic16_dd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_chandra_dd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_track -c 1 -o $O/prof_chandra_dd python tools/one_path.py chandra64 dd > $O/ncu_full.log 2>&1
ls -la $O
