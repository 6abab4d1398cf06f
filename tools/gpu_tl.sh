mkdir -p gpurun_out
for e in grid cluster; do for pr in d dd; do timeout 300 python tools/mgs_timeline.py chandra64 $pr $e; done; done > gpurun_out/timeline.txt 2>&1
timeout 300 python tools/mgs_timeline.py chandra64 qd cluster >> gpurun_out/timeline.txt 2>&1
cat gpurun_out/timeline.txt
for spec in "chandra64 dd 5" "chandra64 d 5" "cyclic16 dd 5"; do
  set -- $spec
  timeout 900 python bench.py --workload $1 --prec $2 --steps $3 --warmup 2 --no-cpu-baseline > gpurun_out/q_$1_$2.json 2> gpurun_out/q_$1_$2.err
done
python tools/show.py
