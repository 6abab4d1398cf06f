O=gpurun_out/r02own; mkdir -p $O
PT_MGS_OWNERS=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "track" > $O/pytest4.log 2>&1; tail -1 $O/pytest4.log
for o in 8 4 2; do for wl in "chandra64 dd 20 5" "chandra64 d 20 5" "cyclic16 dd 10 3"; do set -- $wl
  PT_MGS_OWNERS=$o timeout 600 python bench.py --workload $1 --prec $2 --steps $3 --warmup $4 --no-cpu-baseline > $O/b_$o_$1_$2.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/b_$o_$1_$2.json').read().strip().splitlines()[-1]); print('owners$o $1 $2', round(d['ms_per_step'],2), d.get('critical_path',{}).get('ns_per_column_step'))"
done; done
