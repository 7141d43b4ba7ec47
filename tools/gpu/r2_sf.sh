timeout 900 python -m pytest tests/test_qgemm.py tests/test_parity_shapes.py tests/test_pipeline_gpu.py -m gpu -q -x -k "not production" 2>&1 | tail -2
for s in "20480 5120 3 32" "15360 5120 3 32" "5120 5120 3 32" "5120 20480 3 32"; do
HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so timeout 120 python tools/trace_qgemm.py $s 2>&1 | grep -E "CTAs|final seg|split|exit -" | head -4
done
for v in base prev; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py > gpurun_out/r2_sf.log 2>&1
  echo "$v decode step: $(tail -1 gpurun_out/r2_sf.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_sf_b.log 2>&1
  echo "$v bench: $(grep '^{' gpurun_out/r2_sf_b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"]["sm_mhz"])')"
done
