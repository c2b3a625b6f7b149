cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_metrics.py tests/test_gpu_driver.py -x -q > gpurun_out/t_metrics9.log 2>&1; echo metrics_rc=$?; tail -3 gpurun_out/t_metrics9.log
timeout 300 python tools/bench_configs.py --skip-c5 --configs c3,c4 --iters 20 2>&1 | head -8
