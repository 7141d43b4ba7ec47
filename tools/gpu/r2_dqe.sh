# K3: convert the first slices before waiting for the TMEM A slot (HP_DQ_EARLY=1/2/4) vs default
for v in base dqe1 dqe2 dqe4; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  for b in 3 4 plan; do
    A="--bits $b --per-op"; [ $b = plan ] && A=""
    timeout 600 python tools/decode_step.py $A > gpurun_out/r2_dqe_${v}_$b.log 2>&1
    echo "$v $b: $(tail -1 gpurun_out/r2_dqe_${v}_$b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), round(d["frac_hbm"],3), {k: round(v["us"],1) for k,v in d.get("per_op",{}).items()})')"
  done
done
