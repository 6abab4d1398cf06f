O=gpurun_out/r02s19; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -x -p no:cacheprovider -k "batch" > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
for h in 1 0 1 0; do PT_STREAM_HI=$h timeout 300 python tools/prof_batch.py dd 2368 > $O/prof_h$h.json 2>&1; echo "h$h $(cat $O/prof_h$h.json)"; done
