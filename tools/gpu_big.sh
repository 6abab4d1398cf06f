mkdir -p gpurun_out
timeout 900 python bench.py --workload rand96 --prec dd --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_rand96_dd.json 2> gpurun_out/b_rand96_dd.err
timeout 900 python bench.py --workload cyclic256 --prec qd --steps 1 --warmup 1 --max-steps 2 --no-cpu-baseline > gpurun_out/b_cyclic256_qd.json 2> gpurun_out/b_cyclic256_qd.err
timeout 900 python bench.py --workload batch32 --prec dd --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_batch32_dd.json 2> gpurun_out/b_batch32_dd.err
timeout 900 python bench.py --workload rand96 --prec qd --steps 1 --warmup 1 --max-steps 2 --no-cpu-baseline > gpurun_out/b_rand96_qd.json 2> gpurun_out/b_rand96_qd.err
for f in gpurun_out/b_*.json; do echo $f; head -c 600 $f; echo; done
tail -3 gpurun_out/b_*.err
