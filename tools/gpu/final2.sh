#!/bin/bash
# Round-end check after the decode defaults change: tests, smoke, bench, decode step, prefill ops.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu/final.sh r01c
grep '^{' gpurun_out/bench_r01c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s')}, d['e2e']['value'], d['roofline']['frac'], d['roofline_other']['frac'], d['clocks'])"
VARS="base" bash tools/gpu/dvar2.sh
timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --reps 5 > gpurun_out/r01c_kbench.log 2>&1; echo kbench rc=$?
python -c "
import json
for l in open('gpurun_out/r01c_kbench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
