#!/bin/bash
# iteration loop: GPU parity + quick benches.  SPECS="workload:prec:steps ..."
mkdir -p gpurun_out
rm -f gpurun_out/q_*.json
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider ${PYTEST_K} > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for spec in ${SPECS:-chandra64:dd:5 chandra64:d:5 chandra64:qd:2 cyclic16:dd:5}; do
  IFS=: read -r wl pr st <<< "$spec"
  timeout 600 python bench.py --workload $wl --prec $pr --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/q_${wl}_${pr}.json 2> gpurun_out/q_${wl}_${pr}.err
done
python tools/show.py
