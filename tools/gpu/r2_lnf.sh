timeout 900 python -m pytest tests/test_ln_fold.py tests/test_pipeline_gpu.py tests/test_qgemm.py tests/test_decoder_glue.py -m gpu -q -x 2>&1 | tail -4
timeout 900 python -m pytest tests/test_pipeline_multigpu.py -m gpu -q -x 2>&1 | tail -2
for v in fold nofold; do
  [ $v = nofold ] && export HP_NO_LN_FOLD=1
  timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_$v.log 2>&1; echo "bench $v rc=$?"
  grep '^{' gpurun_out/r2_bench_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), 'K3', round(d['roofline']['frac'],3), 'K4', round(d['roofline_other']['frac'],3), d['attention']['decode_frac_hbm'], d['gpu_launches'], d['clocks'])"
done
