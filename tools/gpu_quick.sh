#!/bin/bash
# parity + quick perf loop
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 120 python tools/microbench.py > gpurun_out/microbench.json 2>&1
for spec in "chandra64 dd 5" "chandra64 d 5" "chandra64 qd 2" "cyclic16 dd 5" ${EXTRA_SPECS}; do
  set -- $spec
  timeout 900 python bench.py --workload $1 --prec $2 --steps $3 --warmup 2 --no-cpu-baseline > gpurun_out/q_$1_$2.json 2> gpurun_out/q_$1_$2.err
done
