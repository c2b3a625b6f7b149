cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or anchors" > gpurun_out/t_fused.log 2>&1; echo fused_rc=$?; tail -30 gpurun_out/t_fused.log
timeout 120 python tools/host_overhead.py
timeout 120 python tools/timeline.py --dim 1000000 --workers 4
timeout 300 python tools/bench_configs.py --skip-c5 --configs c1 --iters 50 2>&1 | head -3
