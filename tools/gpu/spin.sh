#!/bin/bash
# MMA-warp wait variants (spin vs suspend hint) on the 40-layer decode step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
VARS="base _s1 _s3 _s4 base" bash tools/gpu/dvar2.sh
