# round-2 consolidated measurement: GPU tests, smoke, default bench, reference arm, single-path configs
O=gpurun_out/r02final; mkdir -p $O
nvidia-smi -q -d CLOCK > $O/clocks.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_batch32_dd.json 2> $O/bench_batch32_dd.err; tail -c 400 $O/bench_batch32_dd.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_batch32_dd.json 2> $O/bench_reference.err; tail -c 200 $O/bench_reference_batch32_dd.json; echo
for wl in "chandra64 d 20 5" "chandra64 dd 20 5" "cyclic16 dd 10 3" "chandra64 qd 3 3"; do set -- $wl
  timeout 900 python bench.py --workload $1 --prec $2 --steps $3 --warmup $4 > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err
  python -c "import json; d=json.loads(open('$O/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],2), 'ms', d.get('cpu_baseline',{}).get('value'), d.get('cpu_d_all_cores', d.get('cpu_single_thread')))" || tail -2 $O/bench_$1_$2.err
done
timeout 900 python bench.py --workload chandra64 --prec qd --arith fast --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_chandra64_qdfast.json 2>&1
python -c "import json; d=json.loads(open('$O/bench_chandra64_qdfast.json').read().strip().splitlines()[-1]); print('chandra64 qd fast', round(d['ms_per_step'],2))"
timeout 900 python bench.py --workload rand96 --prec dd --max-steps 3 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_rand96_dd_prefix3.json 2>&1
python -c "import json; d=json.loads(open('$O/bench_rand96_dd_prefix3.json').read().strip().splitlines()[-1]); print('rand96 dd prefix3', round(d['ms_per_step'],2))"
