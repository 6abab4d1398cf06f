# SURVEY 8(f) callers on the B200: monodromy degree, Pieri bootstrap, evalbench (Table-9 style reports)
O=gpurun_out/r02callers; mkdir -p $O
for args in "--mode monodromy --cyclic 4 --precision d" "--mode monodromy --cyclic 4 --precision dd" \
            "--mode monodromy --cyclic 16 --precision dd" "--mode pieri --pieri 4,2,2 --precision d" \
            "--mode pieri --pieri 8,4,4 --precision dd" "--mode evalbench --cyclic 16 --reps 100" \
            "--mode track --cyclic 16 --precision dd"; do
  name=$(echo "$args" | tr -d '-' | tr ' ,' '__')
  t0=$(date +%s.%N)
  timeout 900 python -m paper_1501_06625_b200.cli $args > $O/$name.txt 2>&1; rc=$?
  t1=$(date +%s.%N)
  echo "wall_s $(python -c "print(round($t1-$t0,2))") rc=$rc" >> $O/$name.txt
  echo "== $args (rc=$rc)"; tail -6 $O/$name.txt
done
