cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_bench_multirank.py tests/test_gpu_p2p_ipc.py tests/test_gpu_failure.py tests/test_gpu_stress.py -q -p no:cacheprovider 2>&1 | tail -1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['warmup'], d['roofline']['frac'])"
