# memcheck of the single-path and batch engines on the small structured systems
O=gpurun_out/r02san; mkdir -p $O
for ci in 0 1 2 3; do for eng in grid cluster batch; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python tools/repro_random.py $ci $eng > $O/san_${ci}_$eng.txt 2>&1
  echo "case $ci $eng: $(grep -c 'Invalid\|out of bounds' $O/san_${ci}_$eng.txt) findings; $(grep -h 'same\|DIFF\|mismatches\|ERROR' $O/san_${ci}_$eng.txt | tr '\n' ' ')"
done; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
