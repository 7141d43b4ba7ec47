timeout 900 python -m pytest tests/test_k2_indicator.py tests/test_k1_quant.py tests/test_bitplan_chain.py tests/test_capi.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/k12bench.py --shapes 20480x5120,57344x14336 --bits 4 > gpurun_out/r2_k2f.log 2>&1; cut -c1-200 gpurun_out/r2_k2f.log
