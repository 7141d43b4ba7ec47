#!/bin/bash
# Decode ring-depth variants (activation ring 4/5 with deeper code rings) on the 40-layer decode step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
VARS="base _t1 _t2 base" bash tools/gpu/dvar2.sh
