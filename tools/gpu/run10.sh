cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or anchors or cluster" > gpurun_out/t_fused10.log 2>&1; echo fused_rc=$?; tail -3 gpurun_out/t_fused10.log
MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_prof.so timeout 120 python tools/fused_prof.py
timeout 300 python tools/bench_configs.py --skip-c5 --configs c1 --iters 50 2>&1 | head -2
timeout 120 python tools/host_overhead.py
