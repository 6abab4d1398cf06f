mkdir -p gpurun_out
timeout 300 python bench.py --workload chandra64 --prec qd --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_chandra64_qd_w0.json 2> gpurun_out/b_chandra64_qd_w0.err
PT_MGS_WARP=1 timeout 300 python bench.py --workload chandra64 --prec qd --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_chandra64_qd_w1.json 2> gpurun_out/b_chandra64_qd_w1.err
timeout 600 python bench.py --workload batch32 --prec dd --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_batch32_dd.json 2> gpurun_out/b_batch32_dd.err
timeout 600 python bench.py --workload rand96 --prec dd --steps 1 --warmup 1 --max-steps 3 --no-cpu-baseline > gpurun_out/b_rand96_dd.json 2> gpurun_out/b_rand96_dd.err
timeout 900 python bench.py --workload cyclic256 --prec qd --steps 1 --warmup 0 --max-steps 1 --no-cpu-baseline > gpurun_out/b_cyclic256_qd.json 2> gpurun_out/b_cyclic256_qd.err
for f in gpurun_out/b_*.json; do echo "$f $(python -c "
import json,sys
try:
  d=json.load(open('$f')); print(d['config']['workload'], 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],3), 'frac', round(d['roofline']['frac'],4), d['path'], d.get('phase_ms_per_path'))
except Exception as e: print('ERR', open('$f').read()[:200])
")"; done
tail -2 gpurun_out/b_*.err
