# closed planner loop: predicted (latency model -> pipesim) vs measured rounds,
# synthetic-model plans vs plans from the B200-fitted model
timeout 1500 python tools/plan_eval.py opt13b_b32_1gpu opt13b_b32_1gpu_b200lat opt30b_b32_1gpu opt30b_b32_1gpu_b200lat > gpurun_out/r2_plan_eval.log 2>&1; echo "eval rc=$?"
cut -c1-400 gpurun_out/r2_plan_eval.log
for p in opt13b_b32_1gpu_b200lat opt30b_b32_1gpu_b200lat; do
  timeout 900 python bench.py --plan $p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$p.log 2>&1; echo "bench $p rc=$?"
  grep '^{' gpurun_out/r2_bench_$p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["kernel"][:3], d["roofline"]["frac"], d["roofline_other"]["kernel"][:3], d["roofline_other"]["frac"])'
done
