cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/timeline_c5.py 2>&1 | tail -1
MARSIT_COIN_PREFETCH=0 timeout 300 python tools/timeline_c5.py 2>&1 | tail -14
