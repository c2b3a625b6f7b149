cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
export MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_prof.so
timeout 300 python tools/merge_level_prof.py --ranks 8 --iters 50 2>&1 | tail -2
timeout 300 python tools/merge_level_prof.py --ranks 8 --topo torus --iters 50 2>&1 | tail -2
