# decode qkv op prefetches the head of each KV-cache context into L2 (HP_KV_PREFETCH = fraction)
HP_KV_PREFETCH=0.3 timeout 900 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x 2>&1 | tail -1
for f in 0 0.15 0.3 0.5 0 0.15 0.3 0.5; do
  HP_KV_PREFETCH=$f timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_kvpf_$f.log 2>&1
  echo "pf=$f bench: $(grep '^{' gpurun_out/r2_kvpf_$f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["decode_tok_s"]), round(d["prefill_tok_s"]), round(d["roofline"]["frac"],3), d["attention"]["decode_avg_us"], d["clocks"]["sm_mhz"])')"
done
