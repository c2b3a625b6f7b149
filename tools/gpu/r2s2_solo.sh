cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank_emulated.py tests/test_gpu_p2p_ipc.py tests/test_gpu_bench_multirank.py -q -x -k "cluster or grid or emulated or p2p or rank or spread or fused" 2>&1 | tail -2
for i in 1 2; do
  echo -n "G8: "; timeout 120 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
  echo -n "G8 torus: "; timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus --iters 100 2>&1 | tail -1
done
MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_prof.so timeout 300 python tools/merge_level_prof.py --ranks 8 --iters 50 2>&1 | tail -1
