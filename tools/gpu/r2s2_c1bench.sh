cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --config c1 --steps 200 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo rc=$?; tail -c 2500 gpurun_out/bench_c1.json; tail -3 gpurun_out/bench_c1.err
timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config']['l2'])"
