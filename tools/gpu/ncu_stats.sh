cd $GRAFT_REPO_ROOT
python tools/bench_metrics.py > gpurun_out/plain_metrics.log 2>&1 && \
ncu --set full --clock-control none -k regex:decode_stats -s 2 -c 1 -o gpurun_out/stats python tools/bench_metrics.py > gpurun_out/ncu_stats.log 2>&1
echo ncu_rc=$?
cat gpurun_out/plain_metrics.log
