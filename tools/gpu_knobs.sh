# runtime-knob sweep of the single-path engines on one box (no rebuild: same SASS)
O=gpurun_out/r02knobs; mkdir -p $O
for rep in 1 2; do
for env in "PT_MGS_B=4" "PT_MGS_B=1" "PT_MGS_B=2" "PT_MGS_B=8" "PT_MGS_WARP=1" "PT_BS_SMEM=0"; do
  for wl in "chandra64 dd 20" "chandra64 d 20" "cyclic16 dd 10"; do set -- $wl
    f=$O/$(echo $env | tr '=' '_')_$1_$2_$rep.json
    env $env timeout 600 python bench.py --workload $1 --prec $2 --steps $3 --warmup 3 --no-cpu-baseline > $f 2>&1
    python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$env $1 $2 $rep', round(d['ms_per_step'],3), {k: round(v,2) for k,v in d.get('phase_ms_per_path',{}).items()})" 2>&1 | tail -1
  done
done; done
