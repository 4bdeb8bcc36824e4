cd $GRAFT_REPO_ROOT
LFM_TC_EXP=4 timeout 300 python scripts/prof_step.py --iters 2 2>&1 | grep "^\[tc" | tail -4
LFM_TC_EXP=5 timeout 300 python scripts/prof_step.py --iters 1 2>&1 | grep "^\[tc" | tail -2
LFM_TC_EXP=7 timeout 300 python scripts/prof_step.py --iters 1 2>&1 | grep "^\[tc" | tail -2
