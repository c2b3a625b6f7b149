cd $GRAFT_REPO_ROOT
O=gpurun_out/r02full
mkdir -p $O
ARGS="--steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1"
python bench.py $ARGS > $O/plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k "regex:extract_kernel|merge_coop|decode_kernel|coins_kernel" -s 8 -c 4 \
    -o $O/full -f python bench.py $ARGS > $O/ncu_full.log 2>&1
echo ncu_rc=$?
tail -3 $O/ncu_full.log
