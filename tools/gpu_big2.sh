mkdir -p gpurun_out/big
O=gpurun_out/big
timeout 900 python bench.py --workload cyclic256 --prec dd --steps 1 --warmup 1 --max-steps 2 --no-cpu-reference > $O/cyclic256_dd.json 2> $O/cyclic256_dd.err
timeout 900 python bench.py --workload cyclic256 --prec qd --steps 1 --warmup 0 --max-steps 1 --no-cpu-reference > $O/cyclic256_qd.json 2> $O/cyclic256_qd.err
timeout 900 python bench.py --workload rand96 --prec dd --steps 1 --warmup 1 --max-steps 3 --no-cpu-reference > $O/rand96_dd.json 2> $O/rand96_dd.err
timeout 900 python bench.py --workload rand96 --prec qd --steps 1 --warmup 0 --max-steps 1 --no-cpu-reference > $O/rand96_qd.json 2> $O/rand96_qd.err
timeout 900 python bench.py --workload cyclic16 --prec dd > $O/cyclic16_dd.json 2> $O/cyclic16_dd.err
for f in $O/*.json; do python -c "
import json
d=json.load(open('$f'))
c=d.get('cpu_d_all_cores') or {}
print('$f', d['config']['workload'], 'ms', round(d['ms_per_step'],2), 'iters', d['path']['newton_iters'], 'ms/iter', round(1e3*d.get('sec_per_newton_iter',0),3), 'cpuD ms/iter', round(1e3*c.get('sec_per_newton_iter',0),3), 'cpuD ms/path', round(1e3*c.get('sec_per_path',0),2), 'frac', round(d['roofline']['frac'],4), d.get('phase_ms_per_path'))
"; done
