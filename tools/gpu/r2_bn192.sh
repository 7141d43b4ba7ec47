# prefill BN=192 tiles with a double-buffered accumulator (exp bn192) vs BN=256 single accumulator (base)
export HP_LIB_PATH=$PWD/exp/libhetplan_b200_bn192.so
timeout 1200 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py tests/test_pipeline_gpu.py -m gpu -q -x 2>&1 | tail -2
unset HP_LIB_PATH
for v in base bn192; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/kbench.py --op prefill --bits 3,4,16 > gpurun_out/r2_bn192_kb_$v.log 2>&1; echo "$v kbench rc=$?"; tail -14 gpurun_out/r2_bn192_kb_$v.log
done
for v in base bn192 base bn192; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bn192_b_$v.log 2>&1
  echo "$v bench: $(grep '^{' gpurun_out/r2_bn192_b_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["decode_tok_s"]), round(d["prefill_tok_s"]), round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"]["sm_mhz"])')"
done
