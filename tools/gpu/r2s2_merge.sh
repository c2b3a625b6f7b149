cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for k in grid coop; do echo "== $k"; MARSIT_MERGE_KERNEL=$k MARSIT_MERGE_DEBUG=1 timeout 120 python tools/bench_merge.py --iters 50 2>&1 | tail -3; done
for k in grid coop; do echo "== G8 $k"; MARSIT_MERGE_KERNEL=$k timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1; done
for k in grid coop; do echo "== C3 round $k"; MARSIT_MERGE_KERNEL=$k timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -1; done
