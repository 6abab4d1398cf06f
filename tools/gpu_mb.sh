mkdir -p gpurun_out
timeout 120 python tools/microbench.py > gpurun_out/microbench.json 2>&1
for p in d dd qd; do for e in cluster grid; do timeout 300 python tools/mgs_timeline.py chandra64 $p $e >> gpurun_out/timeline.jsonl 2>&1; done; done
cat gpurun_out/microbench.json gpurun_out/timeline.jsonl
