timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_decoder_glue.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_lnrows.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_lnrows.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), 'K3', round(d['roofline']['frac'],3), 'K4', round(d['roofline_other']['frac'],3), d['attention']['decode_frac_hbm'], d['clocks'])"
