# Profiles for profiles/ (one GPU): ncu only after the same command exits 0.
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K3='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(16|32), '
K4='regex:qgemm_kernel<\(int\)[0-9]+, \(bool\)1, \(int\)(128|256), '
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
grep -q '^{' gpurun_out/plain.log || exit 1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "$K3" -c 4 -o gpurun_out/k3_full_r01 $B > gpurun_out/ncu_k3.log 2>&1; echo ncu3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "$K4" -c 4 -o gpurun_out/k4_full_r01 $B > gpurun_out/ncu_k4.log 2>&1; echo ncu4 rc=$?
timeout 300 $B --no-graphs > gpurun_out/plain_eager.log 2>&1; echo plain eager rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r01.csv $B --no-graphs > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
ls -la gpurun_out | grep -E "ncu-rep|csv"
