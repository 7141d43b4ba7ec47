# N=1 bench (OPT-13B configs[1]) incl. cpu_baseline, the reference arm, and
# the north_star target plan (OPT-30B mixed 3/4/8/16 on one B200)
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1.log 2>&1; echo "bench rc=$?"
tail -c 6000 gpurun_out/r2_bench_n1.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
tail -c 3000 gpurun_out/r2_bench_ref.log
timeout 900 python bench.py --plan opt30b_b32_1gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_opt30b.log 2>&1; echo "opt30b rc=$?"
tail -c 4000 gpurun_out/r2_bench_opt30b.log
