export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
for c in 97 134 40; do
  echo "== CTA $c"; HP_QGEMM_TRACE_CTA=$c timeout 120 python tools/trace_qgemm.py 20480 5120 3 32 --roles 2>&1 | grep -vE "^\s*$" | grep -A6 -E "^epilogue|^fixup|slow CTA $c" | head -24
done
