timeout 900 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -k "reference_decoder" -rA 2>&1 | grep -E "PASS|FAIL|Error|assert|passed|failed" | head -12
