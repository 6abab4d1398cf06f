O=gpurun_out/r02s16; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_monodromy.py -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
for u in 1 0 1 0; do PT_UNIFORM=$u timeout 300 python tools/prof_batch.py dd 2368 > $O/prof_u$u.json 2>&1; echo "u$u $(cat $O/prof_u$u.json)"; done
