# locate the stall of test_pipeline_gpu.py run as the first module
timeout 400 python -m pytest "tests/test_pipeline_gpu.py::test_opt125m_round_matches_reference_decoder[False-None-None]" -m gpu -v -x -p no:cacheprovider --timeout 150 --timeout-method thread > gpurun_out/r2_pipehang_b.log 2>&1; echo "eager alone rc=$?"
grep -E "PASSED|FAILED|Timeout|passed|failed" gpurun_out/r2_pipehang_b.log | head -5
grep -B2 -A12 "Timeout" gpurun_out/r2_pipehang_b.log | grep -E "File|line|Thread" | head -40
timeout 400 python -m pytest tests/test_capi.py tests/test_pipeline_gpu.py -m gpu -q -x -p no:cacheprovider --timeout 150 --timeout-method thread > gpurun_out/r2_pipehang_c.log 2>&1; echo "after capi rc=$?"
tail -3 gpurun_out/r2_pipehang_c.log
