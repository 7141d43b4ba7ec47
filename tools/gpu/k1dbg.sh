for v in base k1p0; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "== $v"; timeout 300 python tools/k1_debug.py 2>&1 | tail -40
done
