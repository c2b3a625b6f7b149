cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t16.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/t16.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 300 python bench.py > gpurun_out/b16.json 2> gpurun_out/b16.err; echo bench_rc=$?; cat gpurun_out/b16.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d.get('phases_us'), d['clocks'])"
