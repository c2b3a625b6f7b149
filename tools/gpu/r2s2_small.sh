cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank_emulated.py tests/test_gpu_p2p_ipc.py -q -x -k "cluster or grid or emulated or p2p or rank" 2>&1 | tail -2
for r in 1 2; do for sm in 0 1; do
  echo -n "small=$sm G8: "; MARSIT_GRID_SMALL=$sm MARSIT_MERGE_DEBUG=1 timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | grep -v "^merge" | tail -1
  echo -n "small=$sm G8 torus: "; MARSIT_GRID_SMALL=$sm timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus --iters 100 2>&1 | tail -1
  echo -n "small=$sm G4: "; MARSIT_GRID_SMALL=$sm timeout 120 python tools/bench_merge_rank.py --ranks 4 --iters 100 2>&1 | tail -1
done; done
MARSIT_MERGE_DEBUG=1 timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 10 2>&1 | grep "merge grid" | head -2
MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_prof.so timeout 300 python tools/merge_level_prof.py --ranks 8 --iters 50 2>&1 | tail -1
