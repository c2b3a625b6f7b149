cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 120 python -m pytest tests/test_gpu_failure.py -x -v > gpurun_out/t_failure3.log 2>&1; echo failure_rc=$? ; tail -15 gpurun_out/t_failure3.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_metrics.py tests/test_gpu_multirank_emulated.py -x -q > gpurun_out/t_parity3.log 2>&1; echo parity_rc=$?; tail -5 gpurun_out/t_parity3.log
 timeout 120 python tools/bench_merge.py 2>&1 | tail -1
 MARSIT_MERGE_STAGE=0 timeout 120 python tools/bench_merge.py 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
 for G in 8 2; do timeout 120 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1; done
 for cs in 8 12; do MARSIT_MERGE_CSIZE=$cs timeout 120 python tools/bench_merge.py 2>&1 | tail -1; done
timeout 120 python tools/host_overhead.py
timeout 120 python tools/timeline.py --dim 1000000 --workers 4
timeout 120 python tools/timeline.py
