cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_full.log 2>&1; echo gpu_tests_rc=$?; tail -3 gpurun_out/t_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
