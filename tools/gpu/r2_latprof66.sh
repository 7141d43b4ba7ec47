timeout 3000 python tools/latency_profile.py --preset opt-66b > gpurun_out/r2_latprof_opt-66b.log 2>&1; echo "latprof opt-66b rc=$?"; tail -1 gpurun_out/r2_latprof_opt-66b.log
mkdir -p gpurun_out/plans && cp tests/golden/plans/b200_opt66b.* gpurun_out/plans/
