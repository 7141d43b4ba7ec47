for v in base r80 r88; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  timeout 600 python tools/decode_step.py > gpurun_out/r2_r80.log 2>&1
  echo "$v decode step: $(tail -1 gpurun_out/r2_r80.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_us"],1))')"
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_r80_b.log 2>&1
  echo "$v bench: $(grep '^{' gpurun_out/r2_r80_b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"]["sm_mhz"])')"
done
