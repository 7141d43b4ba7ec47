timeout 300 python -m pytest "tests/test_decoder_glue.py" -m gpu -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -30
