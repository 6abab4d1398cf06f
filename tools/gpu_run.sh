O=gpurun_out/r02final2; mkdir -p $O
timeout 1200 python bench.py > $O/bench_batch32_dd.json 2> $O/bench_batch32_dd.err
python -c "import json; d=json.loads(open('$O/bench_batch32_dd.json').read().strip().splitlines()[-1]); print('batch', round(d['value'],1), round(d['ms_per_step'],1), d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic'])"
for wl in "chandra64 d 20 5" "chandra64 dd 20 5" "cyclic16 dd 10 3" "chandra64 qd 3 3"; do set -- $wl
  timeout 900 python bench.py --workload $1 --prec $2 --steps $3 --warmup $4 > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err
  python -c "import json; d=json.loads(open('$O/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],2), 'ms frac', round(d['roofline']['frac'],5), 'cpu', d.get('cpu_baseline',{}).get('value'))" || tail -2 $O/bench_$1_$2.err
done
timeout 900 python bench.py --workload chandra64 --prec qd --arith fast --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_chandra64_qdfast.json 2>&1
python -c "import json; d=json.loads(open('$O/bench_chandra64_qdfast.json').read().strip().splitlines()[-1]); print('chandra64 qd fast', round(d['ms_per_step'],2))"
for c in 8 4 2; do for wl in "cyclic16 dd" "chandra64 dd"; do set -- $wl
  PT_CLUSTER_MAX=$c timeout 600 python bench.py --workload $1 --prec $2 --steps 5 --warmup 3 --no-cpu-baseline > $O/b_c$c.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/b_c$c.json').read().strip().splitlines()[-1]); print('cluster<=$c $1 $2', round(d['ms_per_step'],2))"
done; done
