#!/bin/bash
# After the proxy-fence fix: full GPU tests, smoke, determinism diag, decode step, prefill ops, bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu/final.sh fix
DIAG_BITS=16,4 timeout 300 python tools/dpsk_diag.py > gpurun_out/fix_diag.log 2>&1; echo "diag rc=$?"; awk '{print $1,$2,$4,$5, $(NF-4), $(NF-3), $(NF-2), $(NF-1), $NF}' gpurun_out/fix_diag.log
VARS="base" bash tools/gpu/dvar2.sh
timeout 600 python tools/kbench.py --op prefill --m-pre 2048 --reps 5 > gpurun_out/fix_kbench.log 2>&1; echo kbench rc=$?
python -c "
import json
for l in open('gpurun_out/fix_kbench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['k'], d['bits'], round(d['us'],1), round(d['TFs']))"
