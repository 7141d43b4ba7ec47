#!/bin/bash
bash tools/gpu/k3check.sh k3nb
timeout 900 python tools/latency_profile.py > gpurun_out/latency_profile.log 2>&1; echo "latency rc=$?"; tail -2 gpurun_out/latency_profile.log
cp tests/golden/plans/b200_opt13b.profile.csv tests/golden/plans/b200_opt13b.latency_model.json gpurun_out/ 2>/dev/null
