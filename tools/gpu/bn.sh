#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_qgemm.py tests/test_pipeline_gpu.py -m gpu -x -q > gpurun_out/bn_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bn_tests.log
timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --bits 3,4 --reps 5 > gpurun_out/kbench_pre_bn.log 2>&1; echo kbench rc=$?
python -c "
import json
for l in open('gpurun_out/kbench_pre_bn.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
timeout 600 python bench.py > gpurun_out/bench_bn.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_bn.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s')}, d['e2e']['value'], d['roofline']['kernel'][:3], d['roofline']['frac'])"
