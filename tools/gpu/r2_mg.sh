# multi-GPU: pipeline parity tests (small + planner OPT-30B partitions) and the bench at N GPUs
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_pipeline_multigpu.py -m gpu -q -rA > gpurun_out/r2_mg_tests_$N.log 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|SKIP|passed|failed|Error" gpurun_out/r2_mg_tests_$N.log | tail -12
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/r2_bench_n$N.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_n$N.log | cut -c1-600
