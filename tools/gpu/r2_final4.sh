# end-of-session check: full GPU suite (driver order), smoke, N=1 bench
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2_final4_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -1 gpurun_out/r2_final4_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_final4_n1.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_final4_n1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["decode_tok_s"]), round(d["prefill_tok_s"]), d["gpu_launches"], round(d["roofline"]["frac"],3), round(d["roofline_other"]["frac"],3), d["clocks"]["sm_mhz"], round(d["cpu_baseline"]["value"],1))'
