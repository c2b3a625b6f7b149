cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or spread or coin" 2>&1 | tail -1
for D in 1000000 250000; do for sp in 1 0; do MARSIT_SPREAD=$sp timeout 120 python tools/spread_probe.py $D 4 2>&1 | tail -1; done; done
MARSIT_STASH=0 MARSIT_SPREAD=0 timeout 120 python tools/spread_probe.py 2>&1 | tail -1
MARSIT_STASH=0 timeout 120 python tools/spread_probe.py 2>&1 | tail -1
for sp in 1 0; do MARSIT_SPREAD=$sp timeout 120 python tools/spread_probe.py 1000000 8 2>&1 | tail -1; done
timeout 300 python tools/bench_configs.py --skip-c5 --configs c1 --iters 200 2>&1 | head -3
timeout 120 python tools/host_overhead.py
