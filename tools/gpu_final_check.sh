O=gpurun_out/r02final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for wl in "chandra64 d 20" "cyclic16 d 10" "chandra64 dd 20"; do set -- $wl
  timeout 600 python bench.py --workload $1 --prec $2 --steps $3 --warmup 3 > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err
  python -c "import json; d=json.loads(open('$O/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],3), d['path']['steps'], d['path']['newton_iters'], d.get('phase_ms_per_path'))"
done
