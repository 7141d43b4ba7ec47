timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2_all_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2_all_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
