cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for i in 1 2; do
for env in "MARSIT_COIN_L1=0" "MARSIT_COIN_L1=1" "MARSIT_MERGE_PREFETCH=0" "MARSIT_MERGE_PREFETCH=2" "MARSIT_MERGE_PREFETCH=3" "MARSIT_MERGE_MASKS=0" "MARSIT_MERGE_STAGE=0"; do
  echo -n "$env G8: "; env $env timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
done; done
