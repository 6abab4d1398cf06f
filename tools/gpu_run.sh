O=gpurun_out/r02ab2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -x -p no:cacheprovider -k "batch" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in cur old hi0 cur old hi0; do
  case $v in old) export PT_LIB_PATH=$PWD/tools/lib_0287fce.so; unset PT_STREAM_HI;; hi0) unset PT_LIB_PATH; export PT_STREAM_HI=0;; *) unset PT_LIB_PATH PT_STREAM_HI;; esac
  timeout 300 python tools/prof_batch.py dd 2368 > $O/prof_$v.json 2>&1; echo "$v $(cat $O/prof_$v.json)"
done
