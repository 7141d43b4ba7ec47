# K1 f32x2 fast path: bit-exact tests, then rates vs the scalar path
timeout 300 python tools/k1_debug.py 2>&1 | tail -14
timeout 900 python -m pytest tests/test_k1_quant.py tests/test_parity_shapes.py -m gpu -q -x -k "k1 or K1 or quant or golden or oracle" 2>&1 | tail -3
HP_LIB_PATH=$PWD/exp/libhetplan_b200_k1p0.so timeout 900 python -m pytest tests/test_k1_quant.py -m gpu -q -x 2>&1 | tail -2
for v in base k1p0; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/k12bench.py --shapes 20480x5120,57344x14336 --bits 3,4,8 > gpurun_out/r2_k1v2_$v.log 2>&1
  echo "k1 $v:"; cut -c1-200 gpurun_out/r2_k1v2_$v.log | head -12
done
