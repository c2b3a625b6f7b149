cd $GRAFT_REPO_ROOT
python tools/bench_merge.py --iters 3 > gpurun_out/plain_c3g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:merge_grid -s 3 -c 1 -o gpurun_out/merge_grid_c3 python tools/bench_merge.py --iters 3 > gpurun_out/ncu_c3g.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_c3g.log
