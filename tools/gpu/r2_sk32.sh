timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x -k "not production" 2>&1 | tail -2
HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so timeout 120 python tools/trace_qgemm.py 20480 5120 3 32 2>&1 | grep -E "CTAs|final|split|lastMMA|exit -" | head -6
for v in base prev; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  for r in 1 2; do
  timeout 600 python tools/decode_step.py > gpurun_out/r2_sk.log 2>&1
  echo "$v decode step: $(tail -1 gpurun_out/r2_sk.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
  done
done
