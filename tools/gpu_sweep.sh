# MGS tuning sweep: cluster size x column block
for C in 16 8 4; do for B in 2 4 8; do
  echo "C=$C B=$B $(PT_CLUSTER_MAX=$C PT_MGS_B=$B python tools/mgs_timeline.py ${1:-chandra64} ${2:-dd} | python -c 'import json,sys; d=json.load(sys.stdin); print(d["total_ns"], {k[:12]: v for k, v in d["per_column_median"].items()})')"
done; done
