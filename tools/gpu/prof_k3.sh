#!/bin/bash
# Refresh the bench-round K3 --set full capture (layer 0's four decode ops) and the
# single-op K3 (3/4/8-bit fc1) + K1/K2 captures with the shipped kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K3='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(16|32), '
timeout 300 $B > gpurun_out/plain_k3.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "$K3" -c 4 -o gpurun_out/k3_full_r01 $B > gpurun_out/ncu_k3.log 2>&1; echo ncu3 rc=$?
bash tools/gpu/ncu_k3.sh r01
