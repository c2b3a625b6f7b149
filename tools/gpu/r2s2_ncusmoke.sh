cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo ncu_smoke_rc=$?
grep -E "smoke:|ERROR|round_spread|==PROF== Profiling" gpurun_out/ncu_smoke.log | sort | uniq -c | head -20
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
