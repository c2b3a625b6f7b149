cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank_emulated.py -q -x -k "fused or spread or coin or emulated" 2>&1 | tail -3
for i in 1 2; do for t in 1 0; do echo -n "tma=$t "; MARSIT_SPREAD_TMA=$t timeout 120 python tools/spread_probe.py 2>&1 | tail -1; done; done
for t in 1 0; do echo -n "M8 tma=$t "; MARSIT_SPREAD_TMA=$t timeout 120 python tools/spread_probe.py 1000000 8 2>&1 | tail -1; done
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
