cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for i in 1 2; do for c in 1 0; do
  echo -n "coop=$c G8: "; MARSIT_GRID_COOP=$c timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
  echo -n "coop=$c C2: "; MARSIT_GRID_COOP=$c timeout 120 python tools/bench_merge.py --dim 61000000 --iters 30 2>&1 | tail -1
done; done
for c in 1 0; do echo "== coop=$c"; MARSIT_GRID_COOP=$c timeout 300 python tools/bench_configs.py --skip-c5 --configs c2 --iters 20 2>&1 | grep -v dense | cut -c1-200; done
