#!/bin/bash
# --set full captures of single decode (K3) qgemm launches at 3/4/8 bits on
# the OPT-13B fc1 shape, plus K1 / K2 launches (one GPU; each ncu run only
# after the same command exits 0 without ncu).
mkdir -p gpurun_out
tag=${1:-r01}
KB="python tools/kbench.py --op decode --shapes 20480x5120 --reps 3"
timeout 300 $KB --bits 3,4,8 > gpurun_out/kbench_dec_$tag.log 2>&1; echo kbench rc=$?
cat gpurun_out/kbench_dec_$tag.log
for b in 3 4 8; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:qgemm_kernel' -s 3 -c 1 -o gpurun_out/k3_b${b}_${tag} $KB --bits $b > gpurun_out/ncu_k3_b$b.log 2>&1; echo ncu k3 b$b rc=$?
done
K12="python tools/k12bench.py --shapes 20480x5120 --bits 4 --reps 1"
timeout 300 $K12 > /dev/null 2>&1; echo k12 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:quant_pack_kernel' -s 2 -c 1 -o gpurun_out/k1_full_$tag $K12 > gpurun_out/ncu_k1.log 2>&1; echo ncu k1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:stats_kernel' -s 2 -c 1 -o gpurun_out/k2_full_$tag $K12 > gpurun_out/ncu_k2.log 2>&1; echo ncu k2 rc=$?
ls -la gpurun_out | grep ncu-rep
