# round 2: new parity tests (benched/target shapes, K1 production sizes,
# K2 -> omega -> plan chain, Theorem-1 K3 check)
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests/test_parity_shapes.py tests/test_theorem1.py tests/test_bitplan_chain.py -m gpu -q -rA --durations=15 > gpurun_out/r2_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r2_parity.log
grep -E "PARITY|passed|failed|Error" gpurun_out/r2_parity.log | tail -150
