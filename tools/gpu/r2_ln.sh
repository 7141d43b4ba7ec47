timeout 600 python -m pytest tests -m gpu -q -x -k "layernorm or glue or pipeline_gpu" 2>&1 | tail -2
for v in base lnold; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  for a in "" "--no-ln"; do
    timeout 600 python tools/decode_step.py $a > gpurun_out/r2_ln.log 2>&1
    echo "$v decode step $a: $(tail -1 gpurun_out/r2_ln.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
  done
done
