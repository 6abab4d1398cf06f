# A/B of prebuilt libraries (abprev/lib_<tag>.so, loaded through PT_LIB_PATH)
# on the single-path lines, interleaved twice on one box
O=gpurun_out/r02ablib; mkdir -p $O
for rep in 1 2; do
  for tag in ${TAGS:-base mono slots}; do
    for wl in "cyclic16 dd 10" "chandra64 dd 20" "cyclic16 d 10" "chandra64 d 20" "rand96 dd 3 --max-steps 3"; do set -- $wl
      f=$O/${tag}_$1_$2_$rep.json
      PT_LIB_PATH=abprev/lib_$tag.so timeout 600 python bench.py --workload $1 --prec $2 --steps $3 --warmup 3 --no-cpu-baseline $4 $5 > $f 2>&1
      python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$tag $1 $2 $rep', round(d['ms_per_step'],3), {k: round(v,2) for k,v in d.get('phase_ms_per_path',{}).items()})" 2>&1 | tail -1
    done
  done
done
if [ -n "$BATCH" ]; then
  for rep in 1 2; do for tag in ${TAGS:-base mono slots}; do
    f=$O/${tag}_batch_$rep.json
    PT_LIB_PATH=abprev/lib_$tag.so timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $f 2>&1
    python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$tag batch $rep', round(d['value'],1), round(d['e2e']['value'],1))" 2>&1 | tail -1
  done; done
fi
