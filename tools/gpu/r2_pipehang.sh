# test_pipeline_gpu.py run alone (it did not finish within 900 s in two runs where it was the first module)
timeout 600 python -m pytest tests/test_pipeline_gpu.py -m gpu -v -x -p no:cacheprovider --timeout 240 -s > gpurun_out/r2_pipehang.log 2>&1; echo "alone rc=$?"
grep -E "PASSED|FAILED|Timeout|ERROR|passed|failed" gpurun_out/r2_pipehang.log | head -20
tail -30 gpurun_out/r2_pipehang.log | cut -c1-200
