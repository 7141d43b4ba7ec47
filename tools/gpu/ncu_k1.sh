#!/bin/bash
mkdir -p gpurun_out
tag=${1:-r01}
K12="python tools/k12bench.py --shapes 20480x5120 --bits 4 --reps 1"
timeout 300 $K12 > /dev/null 2>&1; echo k12 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:quant_pack_kernel' -s 2 -c 1 -o gpurun_out/k1_full_$tag $K12 > gpurun_out/ncu_k1.log 2>&1; echo ncu k1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:stats_kernel' -s 2 -c 1 -o gpurun_out/k2_full_$tag $K12 > gpurun_out/ncu_k2.log 2>&1; echo ncu k2 rc=$?
