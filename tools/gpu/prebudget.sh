#!/bin/bash
# Prefill smem budget variants (deeper weight-code ring) on the four OPT-13B prefill ops at 2048 tokens.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "" _p1 _p2; do
  echo "== lib$v"
  HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200$v.so timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --reps 5 > gpurun_out/pb$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/pb$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
done
