export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
for s in "20480 5120 3 32" "15360 5120 3 32" "5120 5120 3 32" "5120 20480 3 32" "20480 5120 4 32"; do
  echo "== $s"; timeout 120 python tools/trace_qgemm.py $s 2>&1 | grep -vE "^\s*$" | head -8
done
