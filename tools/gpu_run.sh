O=gpurun_out/r02s18; mkdir -p $O
timeout 600 python -m pytest tests/test_qdfast.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for e in 0 1; do
  PT_ENGINE=$e timeout 600 python bench.py --workload chandra64 --prec qd --arith fast --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_qdfast_e$e.json 2> $O/err_$e.txt
  python -c "import json; d=json.loads(open('$O/bench_qdfast_e$e.json').read().strip().splitlines()[-1]); print('engine$e', round(d['ms_per_step'],2), d.get('critical_path',{}).get('ns_per_column_step'), d.get('phases_ms'))" || tail -3 $O/err_$e.txt
done
