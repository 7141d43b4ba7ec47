# decode attention split over 2 CTAs: glue tests, standalone rate, pipeline tests, bench
timeout 900 python -m pytest tests/test_decoder_glue.py tests/test_pipeline_gpu.py -m gpu -q -x 2>&1 | tail -2
for sp in 1 2 3; do echo "split $sp: $(timeout 300 python tools/attn_bench.py --split $sp 2>&1 | tail -1)"; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1d.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_n1d.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["ms_per_step"], d["attention"]["decode_frac_hbm"], d["roofline"]["kernel"][:3], d["roofline"]["frac"], d["roofline_other"]["kernel"][:3], d["roofline_other"]["frac"], d["clocks"])'
