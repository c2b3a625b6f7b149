cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 120 python tools/host_overhead.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c1_launches.csv python tools/host_overhead.py > /dev/null 2>&1; echo ncu_rc=$?
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/c1_launches.csv') if not l.startswith('=='))]
from collections import defaultdict
d=defaultdict(list)
for r in rows:
    if r.get('Metric Name')=='gpu__time_duration.sum': d[r['Kernel Name'][:60]].append(float(r['Metric Value']))
for k,v in d.items(): print(f"{k:60s} n={len(v)} median={sorted(v)[len(v)//2]:.0f} {rows[0].get('Metric Unit','')}")
PY
