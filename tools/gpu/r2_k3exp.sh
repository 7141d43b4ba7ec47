# K3 per-SM breakdown experiments (numerics wrong by design in the variants):
# raw = dequant SHF+LOP3 only; nomma = no tcgen05.mma; noact = no activation
# TMA; all3 = all three removed. Plus the parity suite for the asym fix.
timeout 900 python -m pytest tests/test_parity_shapes.py -m gpu -q -rA > gpurun_out/r2_parity2.log 2>&1
echo "parity rc=$?"; grep -E "passed|failed" gpurun_out/r2_parity2.log | tail -2
grep PARITY gpurun_out/r2_parity2.log | sort -t= -k3 -g | tail -3
for v in base raw nomma noact rawnomma all3; do
  if [ $v = base ]; then unset HP_LIB_PATH; else export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so; fi
  timeout 600 python tools/decode_step.py --bits 3 --per-op > gpurun_out/r2_k3exp_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/r2_k3exp_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"]), {k: round(v["us"],1) for k,v in d["per_op"].items()})')"
done
