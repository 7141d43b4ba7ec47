# B200 latency profiles of the 8-GPU configs' layer shapes (OPT-66B, BLOOM-176B)
for p in opt-66b bloom-176b; do
  timeout 1200 python tools/latency_profile.py --preset $p > gpurun_out/r2_latprof_$p.log 2>&1; echo "latprof $p rc=$?"; tail -1 gpurun_out/r2_latprof_$p.log
done
mkdir -p gpurun_out/plans && cp tests/golden/plans/b200_opt66b.* tests/golden/plans/b200_bloom176b.* gpurun_out/plans/ 2>/dev/null; ls gpurun_out/plans
