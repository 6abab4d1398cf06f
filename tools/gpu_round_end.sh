# end-of-round verification on one B200 (run through gpurun):
#   every GPU test, smoke(), the default bench line and the reference arm
O=gpurun_out/r02end; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_batch32_dd.json 2> $O/bench_batch32_dd.err
python -c "import json; d=json.loads(open('$O/bench_batch32_dd.json').read().strip().splitlines()[-1]); print('batch', round(d['value'],1), round(d['ms_per_step'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4))"
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_batch32_dd.json 2> $O/bench_reference.err
python -c "import json; d=json.loads(open('$O/bench_reference_batch32_dd.json').read().strip().splitlines()[-1]); print('reference', d['value'])"
