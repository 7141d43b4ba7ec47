#!/bin/bash
# N-GPU bench under NCCL P2P channel caps (how many SMs the spinning
# send/recv kernels take away from the persistent GEMM grids)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for ch in default 1 2 4; do
  if [ $ch = default ]; then unset NCCL_MAX_P2P_NCHANNELS; else export NCCL_MAX_P2P_NCHANNELS=$ch; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 \
    bench.py --gpus $N --steps 2 --warmup 3 > gpurun_out/bench_n${N}_ch$ch.log 2>&1; echo "ch=$ch rc=$?"
  grep '^{' gpurun_out/bench_n${N}_ch$ch.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  ', {k:round(d.get(k),1) for k in ('value','decode_tok_s','prefill_tok_s')}, 'K4', round(d['roofline']['achieved'] if 'K4' in d['roofline']['kernel'] else d['roofline_other']['achieved']), 'stage_costs', d['stage_costs_s'])"
done
