timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x -k "not production" 2>&1 | tail -1
for v in base prev base prev; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py > gpurun_out/r2_pf.log 2>&1
  echo "$v decode step: $(tail -1 gpurun_out/r2_pf.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
done
