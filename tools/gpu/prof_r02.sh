#!/bin/bash
# Round-2 profile session (1 GPU). ncu only after the same command exited 0.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K3='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(16|32), '
K4='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(128|256), '
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
grep -q '^{' gpurun_out/plain.log || exit 1
# layer 6 (3-bit) of the first prefill / decode unit: skip layers 0-5 (24 launches)
timeout 900 $NCU -k "$K4" -s 24 -c 4 -o gpurun_out/k4_b3_r02 $B > gpurun_out/ncu_k4.log 2>&1; echo ncu k4 rc=$?
timeout 900 $NCU -k "$K3" -s 24 -c 4 -o gpurun_out/k3_b3_r02 $B > gpurun_out/ncu_k3.log 2>&1; echo ncu k3 rc=$?
timeout 900 $NCU -k 'regex:attn_decode' -s 6 -c 2 -o gpurun_out/attn_dec_r02 $B > gpurun_out/ncu_ad.log 2>&1; echo ncu attn-dec rc=$?
timeout 900 $NCU -k 'regex:attn_prefill' -s 6 -c 1 -o gpurun_out/attn_pre_r02 $B > gpurun_out/ncu_ap.log 2>&1; echo ncu attn-pre rc=$?
# cuBLAS bf16 GEMM: the tensor-pipe counter at the measured-peak reference
G="python -c 'import torch; a=torch.randn(8192,8192,device=\"cuda\",dtype=torch.bfloat16); [torch.matmul(a,a) for _ in range(4)]; torch.cuda.synchronize()'"
timeout 300 bash -c "$G" && timeout 600 ncu --set full --clock-control none -k 'regex:gemm|Kernel' -s 2 -c 1 -o gpurun_out/gemm_cublas_r02 bash -c "$G" > gpurun_out/ncu_gemm.log 2>&1; echo ncu gemm rc=$?
bash tools/gpu/ncu_k1.sh r02
timeout 300 $B --no-graphs > gpurun_out/plain_eager.log 2>&1; echo plain eager rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -c 4000 --log-file gpurun_out/launches_r02.csv $B --no-graphs > gpurun_out/ncu_launch.log 2>&1; echo ncu launches rc=$?
ls -la gpurun_out | grep -E "ncu-rep|csv"
