#!/bin/bash
# Producer / dequant wait variants on the 40-layer decode step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
VARS="base _s5 _s6 base" bash tools/gpu/dvar2.sh
