timeout 1800 python -m pytest tests/test_parity_shapes.py -m gpu -q -rA -k "opt66b or bloom176b" > gpurun_out/r2_pbig.log 2>&1; echo rc=$?
grep -c PARITY gpurun_out/r2_pbig.log; grep -E "passed|failed" gpurun_out/r2_pbig.log | tail -2
grep PARITY gpurun_out/r2_pbig.log | sort -t= -k3 -g | tail -2
