timeout 900 python bench.py > gpurun_out/r2_final_n1.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_final_n1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['gpu_launches'], json.dumps(d['roofline'])[:600])"
for p in opt13b_b32_1gpu_b200lat opt30b_b32_1gpu_b200lat; do
  timeout 900 python bench.py --plan $p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$p.log 2>&1; echo "bench $p rc=$?"
  grep '^{' gpurun_out/r2_bench_$p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["ms_per_step"], d["roofline"]["kernel"][:3], round(d["roofline"]["frac"],3), d["roofline_other"]["kernel"][:3], round(d["roofline_other"]["frac"],3))'
done
