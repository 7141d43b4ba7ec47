#!/bin/bash
# 3-bit K3 capture (layer 10 of the OPT-13B plan, decode) with the end-of-session dequant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K3='regex:qgemm_kernel<\(int\)3, \(bool\)1, \(int\)(16|32), '
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled"
timeout 300 $B > gpurun_out/plain_d.log 2>&1; echo plain rc=$?
grep -q '^{' gpurun_out/plain_d.log || exit 1
timeout 900 $NCU -k "$K3" -s 16 -c 4 -o gpurun_out/k3_b3_r02d $B > gpurun_out/ncu_k3d.log 2>&1; echo ncu k3 rc=$?
ls -la gpurun_out | grep -E "ncu-rep"
