#!/bin/bash
# Round-2 refresh after the head-major KV cache / K1 rewrite (1 GPU). ncu only after the same command exited 0.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
grep -q '^{' gpurun_out/plain.log || exit 1
timeout 900 $NCU -k 'regex:attn_decode' -s 6 -c 2 -o gpurun_out/attn_dec_r02 $B > gpurun_out/ncu_ad.log 2>&1; echo ncu attn-dec rc=$?
timeout 900 $NCU -k 'regex:attn_prefill' -s 6 -c 1 -o gpurun_out/attn_pre_r02 $B > gpurun_out/ncu_ap.log 2>&1; echo ncu attn-pre rc=$?
bash tools/gpu/ncu_k1.sh r02
timeout 300 $B --no-graphs > gpurun_out/plain_eager.log 2>&1; echo plain eager rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -c 4000 --log-file gpurun_out/launches_r02.csv $B --no-graphs > gpurun_out/ncu_launch.log 2>&1; echo ncu launches rc=$?
ls -la gpurun_out | grep -E "ncu-rep|csv"
