#!/bin/bash
# K3 decode per-role trace (3/4-bit fc1) with the HP_QGEMM_TRACE library, then the K4 capture refresh.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for b in 3 4; do
HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200_trace.so timeout 300 python tools/trace_qgemm.py 20480 5120 $b 32 > gpurun_out/trace_fc1_b$b.log 2>&1; echo trace$b rc=$?
done
bash tools/gpu/prof_k4.sh
