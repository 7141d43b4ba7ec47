# N=1: default bench (as the driver runs it), the OPT-30B north-star plan, the reference arm
timeout 900 python bench.py > gpurun_out/r2_final_n1.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_final_n1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), 'gen', round(d['generated_tok_s']), 'K3', round(d['roofline']['frac'],3), 'K4', round(d['roofline_other']['frac'],3), d['attention']['decode_frac_hbm'], d['attention']['prefill_tflops'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --plan opt30b_b32_1gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_final_opt30b.log 2>&1; echo "opt30b rc=$?"
grep '^{' gpurun_out/r2_final_opt30b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), 'K3', round(d['roofline']['frac'],3), 'K4', round(d['roofline_other']['frac'],3), d['attention']['decode_frac_hbm'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_final_ref.log 2>&1; echo "ref rc=$?"
grep '^{' gpurun_out/r2_final_ref.log | cut -c1-400
