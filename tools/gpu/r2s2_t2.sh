cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
echo -n "M16 auto "; timeout 120 python tools/spread_probe.py 640000 16 2>&1 | tail -1
