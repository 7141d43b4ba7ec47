set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gpu_tests0.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench0.log 2>&1
tail -c 3000 gpurun_out/r2_bench0.log
cat gpurun_out/r2_gpu_tests0.log
