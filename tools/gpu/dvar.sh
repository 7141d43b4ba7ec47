#!/bin/bash
# K3 decode variants (stage size / dequant warpgroups) on fc1/qkv/out/fc2 at 3/4/8 bits.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "" _v1 _v2; do
HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200$v.so timeout 300 python tools/kbench.py --op decode --bits 3,4,8 --reps 20 > gpurun_out/dvar$v.log 2>&1; echo "var$v rc=$?"
python -c "
import json
for l in open('gpurun_out/dvar$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d.get('GBs',0)))"
done
