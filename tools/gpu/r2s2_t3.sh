cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or spread or coin" 2>&1 | tail -1
for c in 1 0; do echo -n "coop=$c "; MARSIT_SPREAD_COOP=$c timeout 120 python tools/spread_probe.py 2>&1 | tail -1; done
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
