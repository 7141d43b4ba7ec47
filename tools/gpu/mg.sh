#!/bin/bash
# Multi-GPU session (gpurun --gpus N): multi-stage pipeline tests + the N-GPU bench.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
echo "gpus=$N"
timeout 900 python -m pytest tests/test_pipeline_multigpu.py -m gpu -x -q > gpurun_out/mg_tests_$N.log 2>&1; echo "mg tests rc=$?"; tail -3 gpurun_out/mg_tests_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_n$N.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:d.get(k) for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s','n_gpus')}); print(d.get('pipesim')); print(d.get('e2e'))"
tail -5 gpurun_out/bench_n$N.log
