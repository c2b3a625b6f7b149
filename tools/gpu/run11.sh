cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster_merge" > gpurun_out/t_grid.log 2>&1; echo grid_rc=$?; tail -4 gpurun_out/t_grid.log
export MARSIT_MERGE_KERNEL=grid
MARSIT_MERGE_DEBUG=1 timeout 120 python tools/bench_merge.py 2>&1 | tail -2
timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
timeout 120 python tools/bench_merge.py --dim 61000000 2>&1 | tail -1
timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
for G in 8 4 2; do timeout 120 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1; done
timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus 2>&1 | tail -1
echo "--- coop ---"
unset MARSIT_MERGE_KERNEL
timeout 120 python tools/bench_merge.py --dim 61000000 2>&1 | tail -1
timeout 120 python tools/bench_merge_rank.py --ranks 4 2>&1 | tail -1
