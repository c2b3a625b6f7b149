cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for G in 2 4; do for k in grid coop; do echo -n "G$G $k: "; MARSIT_MERGE_KERNEL=$k timeout 120 python tools/bench_merge_rank.py --ranks $G --iters 100 2>&1 | tail -1; done; done
for k in grid coop; do echo -n "G8 torus $k: "; MARSIT_MERGE_KERNEL=$k timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus --iters 100 2>&1 | tail -1; done
for k in grid coop; do echo "== C3 round $k"; MARSIT_MERGE_KERNEL=$k timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -2; done
for k in grid coop; do echo "== C3 round $k again"; MARSIT_MERGE_KERNEL=$k timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -1; done
