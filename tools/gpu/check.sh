#!/bin/bash
# One GPU-box session: GPU tests, bench, fused decode micro-bench.
# usage (from the repo root): bash tools/gpu/check.sh [tag]
tag=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_$tag.log
timeout 300 python tools/fused_bench.py > gpurun_out/fused_$tag.log 2>&1; echo "fused rc=$?"
tail -5 gpurun_out/fused_$tag.log
