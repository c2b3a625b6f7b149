cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all12.log 2>&1; echo gpu_rc=$?; tail -3 gpurun_out/t_all12.log
timeout 900 python tools/bench_configs.py --iters 20 > gpurun_out/configs12.jsonl 2>&1; echo cfg_rc=$?; grep -E '"c1"|"c5"' gpurun_out/configs12.jsonl | head -4
