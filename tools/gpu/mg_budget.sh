#!/bin/bash
# N-GPU bench at several persistent-grid SM budgets (NCCL P2P channels capped by the executor)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_pipeline_multigpu.py -m gpu -x -q > gpurun_out/mg_tests_$N.log 2>&1; echo "mg tests rc=$?"; tail -2 gpurun_out/mg_tests_$N.log
for b in ${BUDGETS:-140 146}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 \
    bench.py --gpus $N --steps 2 --warmup 3 --sm-budget $b > gpurun_out/bench_n${N}_sm$b.log 2>&1; echo "budget=$b rc=$?"
  grep '^{' gpurun_out/bench_n${N}_sm$b.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r={d['roofline']['kernel'][:2]:d['roofline'], d['roofline_other']['kernel'][:2]:d['roofline_other']}
    print('  ', {k:round(d.get(k),1) for k in ('value','decode_tok_s','prefill_tok_s')}, 'K4', round(r['K4']['achieved']), 'K3', round(r['K3']['achieved']), 'e2e', round(d['e2e']['value']), 'gap', d['pipesim'].get('gap'))"
done
