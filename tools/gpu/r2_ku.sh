for v in base ku4 ku16; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "$v: $(timeout 300 python tools/attn_bench.py 2>&1 | tail -1)"
done
# group-scaled decode (HP_DEC_GS) vs default, and its trace
for v in base gs; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py --bits 3 --per-op > gpurun_out/r2_gs_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/r2_gs_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), round(d["frac_hbm"],3), {k: round(v["us"],1) for k,v in d.get("per_op",{}).items()})')"
done
export HP_LIB_PATH=$PWD/exp/libhetplan_b200_gstrace.so
timeout 300 python tools/trace_qgemm.py 20480 5120 3 32 > gpurun_out/r2_gstrace.log 2>&1; grep -E "CTAs|graph" gpurun_out/r2_gstrace.log
