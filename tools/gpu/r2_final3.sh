# end-of-session: full GPU suite, smoke, N=1 bench (OPT-13B configs[1]) and the OPT-30B target plan
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2_final3_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/r2_final3_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_final3_n1.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_final3_n1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["decode_tok_s"]), round(d["prefill_tok_s"]), round(d["generated_tok_s"]), d["ms_per_step"], round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"])'
timeout 900 python bench.py --plan opt30b_b32_1gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_final3_opt30b.log 2>&1; echo "opt30b rc=$?"
grep '^{' gpurun_out/r2_final3_opt30b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["ms_per_step"], round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3))'
