cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_final.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/t_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['frac'], d['phases_ms_per_step'], d['clocks'], d['e2e']['value'])"
timeout 900 python tools/bench_configs.py --iters 40 > gpurun_out/configs_final.txt 2>&1; echo cfg_rc=$?; cut -c1-160 gpurun_out/configs_final.txt
