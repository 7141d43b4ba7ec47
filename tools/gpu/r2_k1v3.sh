# K1 two threads per group: bit-exact tests, then rates (default depth 2 x 3 CTAs vs depth 3 x 2 CTAs)
timeout 300 python tools/k1_debug.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_k1_quant.py tests/test_parity_shapes.py tests/test_qgemm.py -m gpu -q -x 2>&1 | tail -3
for v in base k1r3; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/k12bench.py --shapes 20480x5120,57344x14336,5120x5120 --bits 3,4,8 > gpurun_out/r2_k1v3_$v.log 2>&1
  echo "k1 $v:"; grep K1 gpurun_out/r2_k1v3_$v.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], d['bits'], d['scheme'], round(d['us'],1), round(d['frac'],3))"
done
