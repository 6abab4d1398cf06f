# round-2 headline: default bench (C5) twice + reference arm
O=gpurun_out/r02head; mkdir -p $O
for i in 1 2; do
  timeout 1200 python bench.py > $O/bench_batch32_dd_$i.json 2> $O/bench_batch32_dd_$i.err
  python -c "import json; d=json.loads(open('$O/bench_batch32_dd_$i.json').read().strip().splitlines()[-1]); print('batch', round(d['value'],1), round(d['ms_per_step'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4), d['clocks'])"
done
timeout 1200 python bench.py --paths-per-step 8192 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_batch32_dd_pp8192.json 2>&1
python -c "import json; d=json.loads(open('$O/bench_batch32_dd_pp8192.json').read().strip().splitlines()[-1]); print('batch pp8192', round(d['value'],1))"
