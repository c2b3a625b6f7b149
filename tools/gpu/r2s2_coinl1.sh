cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for r in 1 2; do for c in 0 1; do
  echo -n "coin_l1=$c G8: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
  echo -n "coin_l1=$c G8 torus: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus --iters 100 2>&1 | tail -1
  echo -n "coin_l1=$c G2: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge_rank.py --ranks 2 --iters 100 2>&1 | tail -1
  echo -n "coin_l1=$c C2: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge.py --dim 61000000 --iters 30 2>&1 | tail -1
done; done
