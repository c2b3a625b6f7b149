cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank_emulated.py -q -x -k "fused or spread or coin or emulated" 2>&1 | tail -1
for i in 1 2; do timeout 120 python tools/spread_probe.py 2>&1 | tail -1; done
MARSIT_SPREAD=0 timeout 120 python tools/spread_probe.py 2>&1 | tail -1
MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_prof.so timeout 120 python tools/spread_prof.py 2>&1 | head -1
timeout 300 python tools/bench_configs.py --skip-c5 --configs c1 --iters 200 2>&1 | head -2
