# decoder glue + full pipeline round + weight loader, then the whole gpu suite
timeout 900 python -m pytest tests/test_decoder_glue.py tests/test_pipeline_gpu.py -m gpu -q -x -rA 2>&1 | tail -40 > gpurun_out/r2_decoder.log
cat gpurun_out/r2_decoder.log
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2_gpu_all.log
cat gpurun_out/r2_gpu_all.log
