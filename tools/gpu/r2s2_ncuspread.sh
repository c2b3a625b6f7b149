cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1 SPREAD_NO_GRAPH=1
for env in "MARSIT_STASH=1" "MARSIT_STASH=0" "MARSIT_SPREAD_COOP=0" "MARSIT_STASH=0 MARSIT_SPREAD_COOP=0"; do
  echo "== $env"
  env $env timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:round_spread -c 5 python tools/spread_probe.py 2>&1 | grep -E "ERROR|duration|eager" | head -8
done
