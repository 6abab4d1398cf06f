#!/bin/bash
# measurement session: default bench (+CPU baselines), reference arm, other configs,
# ncu launch list of the default command and one full ncu capture of the tracker kernel
mkdir -p gpurun_out/s
O=gpurun_out/s
nvidia-smi > $O/nvidia_smi.txt
lscpu > $O/lscpu.txt; nproc > $O/nproc.txt
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python bench.py --prec d > $O/bench_chandra_d.json 2> $O/bench_chandra_d.err
timeout 900 python bench.py --prec qd --steps 3 --cpu-seconds 20 > $O/bench_chandra_qd.json 2> $O/bench_chandra_qd.err
timeout 300 python bench.py --workload cyclic16 --no-cpu-reference > $O/bench_cyclic16_dd.json 2> $O/bench_cyclic16_dd.err
timeout 900 python bench.py --workload batch32 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_batch32_dd.json 2> $O/bench_batch32_dd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_chandra_dd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# (full capture in a separate call: tools/gpu_ncu1.sh; the merge-back limit is 64 MiB)
tail -1 $O/pytest_gpu.log
ls $O
