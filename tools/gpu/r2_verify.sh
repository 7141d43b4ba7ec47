# end-of-round verification: full GPU suite, smoke, reference arm
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2_verify_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2_verify_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_verify_ref.log 2>&1; echo "ref rc=$?"
grep '^{' gpurun_out/r2_verify_ref.log | cut -c1-600
