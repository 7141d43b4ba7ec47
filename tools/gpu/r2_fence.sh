# where the dequant warpgroup's stage time goes: trace with / without the tcgen05 fence before the afull arrive
for v in trace tracenf; do
  export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "=== $v"; timeout 300 python tools/trace_qgemm.py 20480 5120 3 32 2>&1 | grep -E "CTAs|graph b2b|dequant" -A12 | grep -E "CTAs|graph|it= ?[0-9]+ " | head -40
done
unset HP_LIB_PATH
for v in base nofence; do
  [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py --bits 3 --per-op > gpurun_out/r2_nf_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/r2_nf_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), round(d["frac_hbm"],3), {k: round(v["us"],1) for k,v in d.get("per_op",{}).items()})')"
done
