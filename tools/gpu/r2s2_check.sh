cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_head.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/t_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err; echo bench_rc=$?; tail -c 3000 gpurun_out/bench_head.json
timeout 300 python tools/bench_configs.py > gpurun_out/configs_head.txt 2>&1; echo cfg_rc=$?; tail -30 gpurun_out/configs_head.txt
