# 3-bit dequant with 8 instead of 15 shifts per 16 pairs; 8-bit on f32x2 pairs (base) vs previous (exp olddq)
timeout 1200 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py tests/test_pipeline_gpu.py -m gpu -q -x 2>&1 | tail -2
for v in base olddq base olddq; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py > gpurun_out/r2_dq3_ds_$v.log 2>&1
  echo "$v decode step (OPT-13B plan): $(tail -1 gpurun_out/r2_dq3_ds_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1), d.get("frac_hbm", d.get("frac")))')"
  timeout 600 python tools/decode_step.py --bits 3 > gpurun_out/r2_dq3_ds3_$v.log 2>&1
  echo "$v decode step (all 3-bit): $(tail -1 gpurun_out/r2_dq3_ds3_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
  timeout 600 python tools/decode_step.py --bits 8 > gpurun_out/r2_dq3_ds8_$v.log 2>&1
  echo "$v decode step (all 8-bit): $(tail -1 gpurun_out/r2_dq3_ds8_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
done
for v in base olddq; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_dq3_b_$v.log 2>&1
  echo "$v bench: $(grep '^{' gpurun_out/r2_dq3_b_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["decode_tok_s"]), round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"]["sm_mhz"])')"
done
