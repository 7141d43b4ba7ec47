# full GPU suite + N=1 bench with the current defaults
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1c.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_n1c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["ms_per_step"], d["attention"]["decode_frac_hbm"], d["roofline"]["kernel"][:3], d["roofline"]["frac"], d["roofline_other"]["kernel"][:3], d["roofline_other"]["frac"], d["clocks"], d["cpu_baseline"]["value"])'
timeout 900 python bench.py --plan opt30b_b32_1gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_opt30b_c.log 2>&1; echo "opt30b rc=$?"
grep '^{' gpurun_out/r2_bench_opt30b_c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["kernel"][:3], d["roofline"]["frac"], d["roofline_other"]["kernel"][:3], d["roofline_other"]["frac"])'
