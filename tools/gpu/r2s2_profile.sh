# Session-2 evidence: bench line, launch list, ncu --set full of the C3 round
# kernels (cooperative merge default) and of the spread small round at C1.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/prof2
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
ARGS="--steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py $ARGS > $O/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:extract_kernel|merge_coop|decode_kernel|coins_kernel" -s 8 -c 4 \
    -o $O/full -f python bench.py $ARGS > $O/ncu_full.log 2>&1; echo full_rc=$?
python tools/ncu_summary.py $O/full.ncu-rep > $O/ncu_summary.txt 2>&1
python tools/ncu_traffic.py $O/full.ncu-rep > $O/ncu_traffic.json 2>&1
rm -f $O/full.ncu-rep
bash tools/gpu/r2s2_profile_spread.sh
