#!/bin/bash
# Round-end style check on one GPU: GPU tests, smoke(), default bench.
mkdir -p gpurun_out
tag=${1:-final}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_$tag.log | tail -1
