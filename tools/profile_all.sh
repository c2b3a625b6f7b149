#!/bin/bash
# Evidence for profiles/: bench line, ncu launch list, ncu --set full of the
# four round kernels, summaries.  Run on the GPU box from the repo root.
set -u
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
ARGS="--steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py $ARGS > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:extract_kernel|merge_coop|decode_kernel|coins_kernel" -s 8 -c 4 \
    -o $O/full -f python bench.py $ARGS > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/full.ncu-rep > $O/ncu_summary.txt 2>&1
python tools/ncu_traffic.py $O/full.ncu-rep > $O/ncu_traffic.json 2>&1
