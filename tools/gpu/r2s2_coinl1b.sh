cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for c in 0 -1 0 -1; do
  echo -n "coin_l1=$c G8: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
  echo -n "coin_l1=$c C4: "; MARSIT_COIN_L1=$c timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 --iters 30 2>&1 | tail -1
done
for c in 0 -1; do echo "== rounds coin_l1=$c"; MARSIT_COIN_L1=$c timeout 600 python tools/bench_configs.py --configs c2,c4 --iters 20 2>&1 | grep -v dense | cut -c1-180; done
