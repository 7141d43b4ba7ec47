for v in base bn128; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "== $v"; timeout 600 python tools/kbench.py --op prefill --bits 3,4,16 2>&1 | grep -E "^\{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'TFs' in d or 'tflops' in str(d).lower(): print({k:(round(v,3) if isinstance(v,float) else v) for k,v in d.items() if k in ('shape','bits','us','TFs','tflops','PFs','frac')})
"
done
