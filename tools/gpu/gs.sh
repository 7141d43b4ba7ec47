#!/bin/bash
# Group-scaled decode variant: parity tests with the variant library, decode-step timing vs base.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200_gs.so timeout 600 python -m pytest tests/test_qgemm.py -m gpu -x -q > gpurun_out/gs_tests.log 2>&1; echo "gs tests rc=$?"; tail -15 gpurun_out/gs_tests.log
VARS="base _gs" bash tools/gpu/dvar2.sh
