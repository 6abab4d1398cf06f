# single-path engine comparison per workload / precision / arithmetic (tools/engine_probe.py)
O=gpurun_out/r02eng; mkdir -p $O
for wl in "chandra64 qd" "cyclic16 qd" "chandra64 dd" "cyclic16 dd" "chandra64 d"; do set -- $wl
  timeout 600 python tools/engine_probe.py $1 $2 3 2>&1 | tail -1
done
for wl in "chandra64 qd" "cyclic16 qd"; do set -- $wl
  for e in 0 1; do
    PT_ENGINE=$e timeout 600 python bench.py --workload $1 --prec $2 --arith fast --steps 3 --warmup 2 --no-cpu-baseline > $O/f_$1_$e.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/f_$1_$e.json').read().strip().splitlines()[-1]); print('fast $1 engine$e', round(d['ms_per_step'],2))"
  done
done
