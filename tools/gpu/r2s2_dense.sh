cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for cfg in c2 c4; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers --clock-control none -k regex:dense -s 2 -c 1 python tools/dense_probe.py $cfg 2>&1 | grep -E "dense_|duration|bytes|registers|grid_size|warps_active|occupancy"
done
