O=gpurun_out/r02sp; mkdir -p $O
timeout 900 python bench.py --workload chandra64 --prec dd --steps 10 --warmup 3 > $O/bench_chandra64_dd.json 2> $O/err.txt
python -c "import json; d=json.loads(open('$O/bench_chandra64_dd.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), d['cpu_d_all_cores'], d['cpu_baseline']['value'])"
timeout 600 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider 2>&1 | tail -1
