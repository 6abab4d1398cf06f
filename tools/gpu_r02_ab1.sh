# A/B: exact vs fast non-finite dd_norm; ncu of the batch kernel
O=gpurun_out/r02ab1; mkdir -p $O
timeout 300 python -m pytest tests/test_cpp_api.py -q -m gpu -p no:cacheprovider > $O/pytest_cpp.log 2>&1; tail -1 $O/pytest_cpp.log
for v in exact fastnf; do
  if [ $v = fastnf ]; then export PT_LIB_PATH=$PWD/tools/libpathtrack_b200_fastnf.so; else unset PT_LIB_PATH; fi
  timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_batch_$v.json 2> $O/bench_batch_$v.err
  timeout 600 python bench.py --workload chandra64 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_chandra_$v.json 2> $O/bench_chandra_$v.err
done
unset PT_LIB_PATH
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track_batch --launch-skip 1 -c 1 -o /tmp/batchdd python tools/prof_batch.py dd 592 > $O/ncu_batch.log 2>&1
python tools/ncu_summary.py /tmp/batchdd.ncu-rep batch_dd > $O/ncu_full_batch_dd.json
ncu -i /tmp/batchdd.ncu-rep --page raw --csv > $O/ncu_raw_batch_dd.csv 2>/dev/null
ncu -i /tmp/batchdd.ncu-rep --page source --csv > $O/ncu_src_batch_dd.csv 2>/dev/null; gzip -f $O/ncu_src_batch_dd.csv
ncu -i /tmp/batchdd.ncu-rep --page details --csv > $O/ncu_details_batch_dd.csv 2>/dev/null
ls -la $O
