timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py -m gpu -q -x -k "not production" 2>&1 | tail -1
timeout 600 python tools/decode_step.py > gpurun_out/r2_order.log 2>&1; echo "decode step: $(tail -1 gpurun_out/r2_order.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
K4='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(128|256), '
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "$K4" -s 24 -c 4 -o gpurun_out/k4_b3_r02 $B > gpurun_out/ncu_k4.log 2>&1; echo ncu k4 rc=$?
