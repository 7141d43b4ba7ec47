#!/bin/bash
# K3/K4 capture refresh with the end-of-round kernels (fast final reduction, shortest-first stream-K order)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K3='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(16|32), '
K4='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(128|256), '
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
grep -q '^{' gpurun_out/plain.log || exit 1
timeout 900 $NCU -k "$K4" -s 24 -c 4 -o gpurun_out/k4_b3_r02 $B > gpurun_out/ncu_k4.log 2>&1; echo ncu k4 rc=$?
timeout 900 $NCU -k "$K3" -s 24 -c 4 -o gpurun_out/k3_b3_r02 $B > gpurun_out/ncu_k3.log 2>&1; echo ncu k3 rc=$?
timeout 300 $B --no-graphs > gpurun_out/plain_eager.log 2>&1; echo plain eager rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -c 4000 --log-file gpurun_out/launches_r02.csv $B --no-graphs > gpurun_out/ncu_launch.log 2>&1; echo ncu launches rc=$?
ls -la gpurun_out | grep -E "ncu-rep|csv"
