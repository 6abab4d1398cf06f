# round 2: GPU tests after the restructure + the default chandra64 DD timing
O=gpurun_out/r02t1; mkdir -p $O
nproc > $O/nproc.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=25 > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/bench_chandra64_dd.json 2> $O/bench_chandra64_dd.err
timeout 600 python bench.py --workload batch32 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_batch32.json 2> $O/bench_batch32.err
tail -c 600 $O/bench_chandra64_dd.json; echo; tail -c 400 $O/bench_batch32.json
