#!/bin/bash
# K3 change check: parity tests, decode micro-benches, N=1 bench
mkdir -p gpurun_out
tag=${1:-k3}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kbench.py --op decode --shapes 15360x5120,5120x5120,20480x5120,5120x20480 --bits 3,4,8 --reps 10 > gpurun_out/kbench_$tag.log 2>&1; echo "kbench rc=$?"
python -c "
import json
for l in open('gpurun_out/kbench_$tag.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['GBs']))"
timeout 300 python tools/fused_bench.py --per-op > gpurun_out/fused_$tag.log 2>&1; echo "fused rc=$?"; cat gpurun_out/fused_$tag.log | tail -1
timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_$tag.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s')}, d['e2e']['value'], d['roofline']['kernel'][:3], d['roofline']['frac'], d['roofline_other']['frac'])"
