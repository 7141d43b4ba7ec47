#!/bin/bash
# Refresh the bench-round K4 --set full capture (layer 0's four prefill ops)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K4='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(128|256), '
timeout 300 $B > gpurun_out/plain_k4.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "$K4" -c 4 -o gpurun_out/k4_full_r01 $B > gpurun_out/ncu_k4.log 2>&1; echo ncu4 rc=$?
