timeout 1200 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x -k "not production" 2>&1 | tail -3
for v in base nossa; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "== $v"; timeout 600 python tools/kbench.py --op prefill --bits 3,4,16 2>&1 | grep -E "^\{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'TFs' in d: print(d.get('shape'), d['bits'], round(d['us'],1), round(d['TFs']))
"
done
