# per-CTA entry/exit spread and CTA-0 role timeline of single decode launches
export HP_LIB_PATH=$PWD/exp/libhetplan_b200_trace.so
for shp in "5120 5120 3" "20480 5120 3" "5120 20480 3"; do
  echo "=== n k bits = $shp"
  timeout 300 python tools/trace_qgemm.py $shp 32 2>&1 | head -120
done > gpurun_out/r2_trace.log 2>&1
grep -E "===|CTAs|graph b2b|exit sorted" gpurun_out/r2_trace.log
