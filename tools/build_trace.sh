#!/bin/bash
# Build libhetplan_b200_trace.so (HP_QGEMM_TRACE) next to the normal library;
# load it with HP_LIB_PATH=.../libhetplan_b200_trace.so (tools/trace_qgemm.py).
set -e
cd "$(dirname "$0")/.."
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2403_01136_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b)'
HP_NVCC_EXTRA="-DHP_QGEMM_TRACE" python -c "$B; b.build(force=True)"
cp paper_2403_01136_b200/libhetplan_b200.so paper_2403_01136_b200/libhetplan_b200_trace.so
python -c "$B; b.build(force=True, verbose=True)"
