export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
HP_QGEMM_TRACE_CTA=10 timeout 120 python tools/trace_qgemm.py 20480 5120 3 2048 --roles 2>&1 | grep -vE "^\s*$" | grep -E "CTAs|exit -|graph|^mma|^epilogue|it=" | head -80
