# test_pipeline_gpu.py as the first module: default (lazy) module loading vs CUDA_MODULE_LOADING=EAGER
export HP_PIPELINE_TIMEOUT_S=45
for i in 1 2 3; do
  for ml in LAZY EAGER; do
    CUDA_MODULE_LOADING=$ml timeout 200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_lazy_${ml}_$i.log 2>&1; rc=$?
    echo "iter $i $ml rc=$rc: $(grep -E 'passed|failed' gpurun_out/r2_lazy_${ml}_$i.log | tail -1) $(grep -oE 'stuck at unit \([a-z]+ [0-9]+ token [0-9]+\)' gpurun_out/r2_lazy_${ml}_$i.log | head -1)"
  done
done
