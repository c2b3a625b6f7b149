cd $GRAFT_REPO_ROOT
python tools/bench_merge_rank.py --ranks 8 --iters 3 > gpurun_out/plain_g8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:merge_cluster -s 3 -c 1 -o gpurun_out/merge_g8 python tools/bench_merge_rank.py --ranks 8 --iters 3 > gpurun_out/ncu_g8.log 2>&1
echo ncu_rc=$?
tail -5 gpurun_out/ncu_g8.log
