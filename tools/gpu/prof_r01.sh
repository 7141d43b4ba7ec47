#!/bin/bash
# Round profile session (1 GPU): K1/K2 --set full captures, then the bench
# round's K3/K4 captures and launch list (tools/prof_round.sh).
cd $GRAFT_REPO_ROOT
bash tools/gpu/ncu_k1.sh r01
bash tools/prof_round.sh
