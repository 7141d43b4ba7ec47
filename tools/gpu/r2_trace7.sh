export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
HP_QGEMM_TRACE_CTA=10 timeout 120 python tools/trace_qgemm.py 20480 5120 3 32 --roles 2>&1 | grep -vE "^\s*$" | grep -A30 -E "^mma|^dequant w4 \(|^dequant w4 detail|^producer" | head -120
