#!/bin/bash
# K3 decode-step variants: 40-layer OPT-13B decode step (per-op launches, graph replay, weights >> L2)
# at the bench plan and uniform 3/4/8 bits, per library variant.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in ${VARS:-"" _v1 _v3 _v4 _v5}; do
  [ "$v" = base ] && v=""
  for b in plan 3 4 8; do
    if [ $b = plan ]; then A=""; else A="--bits $(python -c "print(','.join(['$b']*40))")"; fi
    HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200${v}.so timeout 300 python tools/fused_bench.py --per-op --reps 10 $A > gpurun_out/dstep${v}_${b}.log 2>&1
    echo "var${v} bits=$b rc=$? $(grep '^{' gpurun_out/dstep${v}_${b}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["per_op_graph_us"]), "us", round(d["per_op_GBs"]), "GB/s")')"
  done
done
