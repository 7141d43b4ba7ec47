# B200 latency profiles with the end-of-round kernels (OPT-13B, OPT-30B, OPT-66B, BLOOM-176B layer shapes)
for p in opt-13b opt-30b opt-66b bloom-176b; do
  timeout 1500 python tools/latency_profile.py --preset $p > gpurun_out/r2_latprof_$p.log 2>&1; echo "latprof $p rc=$?"; tail -1 gpurun_out/r2_latprof_$p.log
done
mkdir -p gpurun_out/plans && cp tests/golden/plans/b200_opt13b.* tests/golden/plans/b200_opt30b.* tests/golden/plans/b200_opt66b.* tests/golden/plans/b200_bloom176b.* gpurun_out/plans/ 2>/dev/null; ls gpurun_out/plans
