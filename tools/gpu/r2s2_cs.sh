cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for i in 1 2; do for cs in 4 8 16; do echo -n "cs=$cs "; MARSIT_SPREAD_CSIZE=$cs timeout 120 python tools/spread_probe.py 2>&1 | tail -1; done; done
for cs in 4 8; do echo -n "M8 cs=$cs "; MARSIT_SPREAD_CSIZE=$cs timeout 120 python tools/spread_probe.py 1000000 8 2>&1 | tail -1; done
for cs in 4 8; do echo -n "M16 cs=$cs "; MARSIT_SPREAD_CSIZE=$cs timeout 120 python tools/spread_probe.py 640000 16 2>&1 | tail -1; done
echo -n "M16 KF "; MARSIT_SPREAD=0 timeout 120 python tools/spread_probe.py 640000 16 2>&1 | tail -1
