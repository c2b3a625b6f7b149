cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_all8.log 2>&1; echo all_rc=$?; tail -8 gpurun_out/t_all8.log
timeout 400 python tools/bench_configs.py --skip-c5 --iters 30 > gpurun_out/configs8.jsonl 2>&1; echo configs_rc=$?; head -12 gpurun_out/configs8.jsonl
