# single-pass decode attention + K1 at 4 CTAs/SM: glue/K1 tests, full bench, cuBLAS tensor-counter capture
timeout 900 python -m pytest tests/test_decoder_glue.py tests/test_pipeline_gpu.py tests/test_k1_quant.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1b.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_n1b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["ms_per_step"], d["attention"], d["roofline"]["kernel"][:3], d["roofline"]["frac"], d["roofline_other"]["kernel"][:3], d["roofline_other"]["frac"], d["clocks"])'
G="python -c 'import torch; a=torch.randn(8192,8192,device=\"cuda\",dtype=torch.bfloat16); [torch.matmul(a,a) for _ in range(4)]; torch.cuda.synchronize()'"
timeout 300 bash -c "$G" && timeout 600 ncu --set full --clock-control none -k 'regex:nvjet|gemm' -s 2 -c 1 -o gpurun_out/gemm_cublas_r02 bash -c "$G" > gpurun_out/ncu_gemm.log 2>&1; echo ncu gemm rc=$?
