O=gpurun_out/r02s13; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python tools/prof_batch.py dd 2368 > $O/prof_batch.json 2>&1; cat $O/prof_batch.json
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 1200 $O/bench_default.json
