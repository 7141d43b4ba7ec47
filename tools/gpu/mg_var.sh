#!/bin/bash
# N-GPU bench variants (NCCL env) with per-rank instrumented kernel times
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
export HP_BENCH_PER_RANK=1
run() {
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29520 \
    bench.py --gpus $N --steps 2 --warmup 3 > gpurun_out/bench_n${N}_$tag.log 2>&1; echo "$tag rc=$?"
  grep '^{' gpurun_out/bench_n${N}_$tag.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  ', {k:round(d.get(k),1) for k in ('value','decode_tok_s','prefill_tok_s')})"
  grep '^\[rank' gpurun_out/bench_n${N}_$tag.log | sort
}
run ch2 NCCL_MAX_P2P_NCHANNELS=2
run ch1 NCCL_MAX_P2P_NCHANNELS=1
run ce NCCL_P2P_USE_CUDA_MEMCPY=1
