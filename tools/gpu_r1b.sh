#!/bin/bash
# session re-entry: parity + benches of the current code, both engines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for spec in "chandra64 dd 5" "chandra64 d 5" "chandra64 qd 2" "cyclic16 dd 5" ${EXTRA_SPECS}; do
  set -- $spec
  timeout 600 python bench.py --workload $1 --prec $2 --steps $3 --warmup 3 --no-cpu-baseline > gpurun_out/q_$1_$2.json 2> gpurun_out/q_$1_$2.err
done
python tools/show.py
