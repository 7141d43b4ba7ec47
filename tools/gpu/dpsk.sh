#!/bin/bash
# Prefill data-parallel + stream-K: parity, standalone prefill per op for DP waves 0 (pure stream-K) / default, bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_qgemm.py tests/test_pipeline_gpu.py -m gpu -x -q > gpurun_out/dpsk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dpsk_tests.log
for w in 0 default; do
  if [ $w = default ]; then unset HP_PREFILL_DP_WAVES; else export HP_PREFILL_DP_WAVES=$w; fi
  timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --shapes 5120x5120,5120x20480 --reps 5 > gpurun_out/dpsk_kb_$w.log 2>&1; echo "kbench dp=$w rc=$?"
  python -c "
import json
for l in open('gpurun_out/dpsk_kb_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
done
unset HP_PREFILL_DP_WAVES
timeout 600 python bench.py > gpurun_out/dpsk_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/dpsk_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
