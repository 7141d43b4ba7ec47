# K3 decode with two co-resident half-SM CTAs per SM (HP_DEC_CORES) vs the default
export HP_LIB_PATH=$PWD/exp/libhetplan_b200_cores.so
timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x 2>&1 | tail -3
for v in base cores; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  for b in 3 4 plan; do
    A="--bits $b --per-op"; [ $b = plan ] && A=""
    timeout 600 python tools/decode_step.py $A > gpurun_out/r2_cores_${v}_$b.log 2>&1
    echo "$v $b: $(tail -1 gpurun_out/r2_cores_${v}_$b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), round(d["frac_hbm"],3), {k: round(v["us"],1) for k,v in d.get("per_op",{}).items()})')"
  done
done
# K1 occupancy: 3 CTAs x 256 threads (76 regs) vs 4 CTAs (61 regs)
for v in base k1c4; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/k12bench.py --shapes 20480x5120,57344x14336 --bits 3,4,8 > gpurun_out/r2_k1_$v.log 2>&1
  echo "k1 $v:"; cut -c1-220 gpurun_out/r2_k1_$v.log | head -12
done
