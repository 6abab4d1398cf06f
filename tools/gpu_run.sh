O=gpurun_out/r02cpp; mkdir -p $O
timeout 600 python -m pytest tests/test_cpp_api.py tests/test_bench_contract.py -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
