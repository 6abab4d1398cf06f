# racecheck / synccheck of every engine on small structured systems, memcheck on the pinned workloads
O=gpurun_out/r02san2; mkdir -p $O
for tool in racecheck synccheck; do for ci in 1 4; do for eng in grid cluster batch; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 3 python tools/repro_random.py $ci $eng > $O/${tool}_${ci}_$eng.txt 2>&1
  echo "$tool case $ci $eng: $(grep -h 'same\|DIFF\|mismatches\|ERROR' $O/${tool}_${ci}_$eng.txt | tr '\n' ' ')"
done; done; done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 3 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.txt 2>&1; echo "memcheck smoke: $(tail -2 $O/memcheck_smoke.txt | tr '\n' ' ')"
for ci in 0 1; do for eng in grid cluster batch; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python tools/repro_random.py $ci $eng > $O/memcheck_${ci}_$eng.txt 2>&1
  echo "memcheck case $ci $eng: $(grep -h 'same\|DIFF\|mismatches\|ERROR' $O/memcheck_${ci}_$eng.txt | tr '\n' ' ')"
done; done
