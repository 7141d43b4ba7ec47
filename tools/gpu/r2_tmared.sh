# K3: straggler reduction of the CTA's final segment by bulk copies into the idle activation ring
export HP_LIB_PATH=$PWD/exp/libhetplan_b200_tmared.so
timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x -k "decode or m or benched" 2>&1 | tail -2
for v in base tmared; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  for b in 3 4 plan; do
    A="--bits $b --per-op"; [ $b = plan ] && A=""
    timeout 600 python tools/decode_step.py $A > gpurun_out/r2_tr_${v}_$b.log 2>&1
    echo "$v $b: $(tail -1 gpurun_out/r2_tr_${v}_$b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), round(d["frac_hbm"],3), {k: round(v["us"],1) for k,v in d.get("per_op",{}).items()})')"
  done
done
