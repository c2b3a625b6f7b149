cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for b in 0 2 0 2; do echo -n "balance=$b: "; MARSIT_MERGE_BALANCE=$b timeout 120 python tools/bench_merge.py --iters 50 2>&1 | tail -1; done
for b in 0 2; do echo "== round balance=$b"; MARSIT_MERGE_BALANCE=$b timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -1 | cut -c1-200; done
for b in 0 2; do echo "== round balance=$b"; MARSIT_MERGE_BALANCE=$b timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -1 | cut -c1-200; done
