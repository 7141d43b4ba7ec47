#!/bin/bash
# K1/K2 parity tests + micro-bench, then the pipeline tests and the N=1 bench.
mkdir -p gpurun_out
tag=${1:-a}
timeout 600 python -m pytest tests/test_k1_quant.py tests/test_k2_indicator.py tests/test_dropin.py -m gpu -x -q > gpurun_out/k12_tests_$tag.log 2>&1; echo "k12 tests rc=$?"; tail -3 gpurun_out/k12_tests_$tag.log
timeout 600 python tools/k12bench.py > gpurun_out/k12bench_$tag.log 2>&1; echo "k12bench rc=$?"
python - <<'P'
import json,sys
for l in open(sys.argv[1] if len(sys.argv)>1 else "gpurun_out/k12bench_TAG.log".replace("TAG", __import__("os").environ.get("TAG","a"))):
    if l.startswith("{"):
        d=json.loads(l)
        if "summary" in d: print(d); continue
        print(d["kernel"], d["shape"], d.get("bits",""), d.get("scheme",""), round(d["us"],1), round(d["GBs"]), round(d["frac"],3))
P
if [ "$2" = "full" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
  timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$tag.log
fi
