# K3 tail experiments + B200 latency profiles (OPT-13B, OPT-30B layers incl. attention)
for v in base nored tiles; do
  unset HP_LIB_PATH HP_EXP_DECODE_TILES
  [ $v = nored ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_nored.so
  [ $v = tiles ] && export HP_EXP_DECODE_TILES=1
  timeout 600 python tools/decode_step.py --bits 3 --per-op > gpurun_out/r2_k3exp2_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/r2_k3exp2_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), {k: round(v["us"],1) for k,v in d["per_op"].items()})')"
done
unset HP_LIB_PATH HP_EXP_DECODE_TILES
for p in opt-13b opt-30b; do
  timeout 900 python tools/latency_profile.py --preset $p > gpurun_out/r2_latprof_$p.log 2>&1; echo "latprof $p rc=$?"; tail -1 gpurun_out/r2_latprof_$p.log
done
mkdir -p gpurun_out/plans && cp tests/golden/plans/b200_opt13b.* tests/golden/plans/b200_opt30b.* gpurun_out/plans/ 2>/dev/null; ls gpurun_out/plans
