#!/bin/bash
# K4 weight-major tile walk: parity tests, standalone prefill per op, bench, DRAM bytes per launch.
mkdir -p gpurun_out
tag=${1:-wm}
timeout 900 python -m pytest tests/test_qgemm.py tests/test_pipeline_gpu.py -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --reps 5 > gpurun_out/${tag}_kbench.log 2>&1; echo kbench rc=$?
python -c "
import json
for l in open('gpurun_out/${tag}_kbench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/${tag}_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','decode_tok_s','prefill_tok_s')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qgemm --csv \
  --log-file gpurun_out/${tag}_ncu_dram.csv python tools/kbench.py --op prefill --m-pre 2048 --bits 3,4,16 --reps 1 --no-flush > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"
