# head-major KV cache: glue + pipeline tests, attention split sweep, bench
timeout 900 python -m pytest tests/test_decoder_glue.py tests/test_pipeline_gpu.py tests/test_pipeline_multigpu.py -m gpu -q -x 2>&1 | tail -3
for s in 1 2; do timeout 120 python tools/attn_bench.py --p 560 --split $s; done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_hm.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/r2_bench_hm.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), d['attention'], round(d['roofline']['frac'],3), round(d['roofline_other']['frac'],3), d['clocks'])"
