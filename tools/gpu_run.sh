O=gpurun_out/r02p2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_monodromy.py -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in cur prev cur prev; do
  case $v in prev) export PT_LIB_PATH=$PWD/tools/lib_prev.so;; *) unset PT_LIB_PATH;; esac
  timeout 300 python tools/prof_batch.py dd 2368 > $O/p_$v.json 2>&1; echo "$v $(cat $O/p_$v.json)"
done
for v in cur prev; do
  case $v in prev) export PT_LIB_PATH=$PWD/tools/lib_prev.so;; *) unset PT_LIB_PATH;; esac
  timeout 600 python bench.py --workload cyclic16 --prec dd --steps 10 --warmup 3 --no-cpu-baseline > $O/c_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/c_$v.json').read().strip().splitlines()[-1]); print('cyclic16 dd $v', round(d['ms_per_step'],2))"
done
