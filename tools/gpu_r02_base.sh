# round-2 baseline: GPU tests, batch phase profile, ncu full captures of the
# throughput kernels (k_track_batch, k_track_grid on rand96 / cyclic256)
O=gpurun_out/r02base; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python tools/prof_batch.py dd 2368 > $O/prof_batch_dd.json 2>&1
ncap() {  # name, command...
  local name=$1; shift
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track -c 1 -o /tmp/$name "$@" > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep $name > $O/ncu_full_$name.json
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/ncu_raw_$name.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv > $O/ncu_src_$name.csv 2>/dev/null
  gzip -f $O/ncu_src_$name.csv
}
ncap batch_dd python tools/prof_batch.py dd 296
ncap rand96_dd python tools/one_prefix.py rand96 dd 1
ncap rand96_qd python tools/one_prefix.py rand96 qd 0
ncap cyclic256_qd python tools/one_prefix.py cyclic256 qd 0
ls -la $O
