#!/bin/bash
mkdir -p gpurun_out
tag=${1:-c}
timeout 600 python -m pytest tests/test_k1_quant.py tests/test_k2_indicator.py -m gpu -x -q > gpurun_out/k12_tests_$tag.log 2>&1; echo "k12 tests rc=$?"; tail -2 gpurun_out/k12_tests_$tag.log
timeout 600 python tools/k12bench.py --shapes 20480x5120,57344x14336 > gpurun_out/k12bench_$tag.log 2>&1; echo "k12bench rc=$?"
grep -v summary gpurun_out/k12bench_$tag.log | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['kernel'], d['shape'], d.get('bits',''), d.get('scheme',''), round(d['us'],1), round(d['GBs']), round(d['frac'],3))"
for b in ${TRACEBITS:-}; do
HP_LIB_PATH=$PWD/paper_2403_01136_b200/libhetplan_b200_trace.so timeout 120 python tools/trace_qgemm.py 20480 5120 $b 32 > gpurun_out/trace_qgemm_b$b.log 2>&1; echo trace rc=$?
head -60 gpurun_out/trace_qgemm_b$b.log
done
