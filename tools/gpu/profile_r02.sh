cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python bench.py --dtype f64 --no-cpu-baseline > $O/bench_f64.json 2> $O/bench_f64.err; echo f64_rc=$?
python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1_rc=$?
python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref_rc=$?
ARGS="--steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1"
python bench.py $ARGS > $O/plain_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py $ARGS > $O/ncu_launches.log 2>&1; echo ncu_rc=$?
cat $O/bench.json
