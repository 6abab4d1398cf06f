# end-of-round verification on one B200 (run through gpurun):
#   every GPU test, smoke(), the default bench line, the reference arm, the single-path lines
O=gpurun_out/r02end4; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_batch32_dd.json 2> $O/bench_batch32_dd.err
python -c "import json; d=json.loads(open('$O/bench_batch32_dd.json').read().strip().splitlines()[-1]); print('batch', round(d['value'],1), round(d['ms_per_step'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4))"
for wl in "chandra64 qd 3 3" "chandra64 dd 20 5"; do set -- $wl
  timeout 900 python bench.py --workload $1 --prec $2 --steps $3 --warmup $4 > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err
  python -c "import json; d=json.loads(open('$O/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],2), d['path']['steps'], d['path']['newton_iters'], round(d['roofline']['frac'],5))"
done
timeout 900 python bench.py --workload chandra64 --prec qd --arith fast --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_chandra64_qdfast.json 2>&1
python -c "import json; d=json.loads(open('$O/bench_chandra64_qdfast.json').read().strip().splitlines()[-1]); print('chandra64 qd fast', round(d['ms_per_step'],2))"
timeout 900 python bench.py --impl reference > $O/bench_reference_batch32_dd.json 2> $O/bench_reference.err
python -c "import json; d=json.loads(open('$O/bench_reference_batch32_dd.json').read().strip().splitlines()[-1]); print('reference', round(d['value'],2), d['cpu_baseline']['sample'])"
