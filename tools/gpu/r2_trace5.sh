export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
timeout 120 python tools/trace_qgemm.py 5120 5120 3 32 2>&1 | grep -E "CTAs|final seg|split|exit -|slow CTA" | head -12
