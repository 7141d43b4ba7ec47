#!/bin/bash
# 16-bit prefill stream-K race: determinism diagnostic per candidate-fix library.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "" _f1 _f2 _f3; do
  echo "== lib$v"
  DIAG_BITS=16 HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200$v.so timeout 300 python tools/dpsk_diag.py 2>&1 | grep -v "^$" | awk '{print $1,$2,$5,$6,$NF, $(NF-1), $(NF-2), $(NF-3), $(NF-4)}'
done
