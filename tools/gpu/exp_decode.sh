#!/bin/bash
# Decode (K3 fused) experiments: per-bit fused vs per-op, and a per-op trace.
mkdir -p gpurun_out
out=gpurun_out/exp_decode_${1:-a}.log
: > $out
for b in 3 4 8 16; do
  bits=$(python -c "print(','.join(['$b']*40))")
  timeout 300 python tools/fused_bench.py --bits $bits --per-op >> $out 2>&1
done
timeout 300 python tools/fused_bench.py --per-op >> $out 2>&1
for b in 3 4; do
  HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200_dtrace.so timeout 120 python tools/trace_dstage.py $b 2 >> $out 2>&1
done
timeout 600 python tools/k12bench.py >> $out 2>&1
cat $out | grep -v "^  op\|epi_done by" | head -150
