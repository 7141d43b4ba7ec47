export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
for c in 29 118; do
  echo "== CTA $c"; HP_QGEMM_TRACE_CTA=$c timeout 120 python tools/trace_qgemm.py 5120 5120 3 32 --roles 2>&1 | grep -vE "^\s*$" | grep -A8 -E "^epilogue|^fixup|^mma" | head -40
done
