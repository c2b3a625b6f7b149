cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or anchors or golden" > gpurun_out/t_parity5.log 2>&1; echo parity_rc=$?; tail -5 gpurun_out/t_parity5.log
timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
MARSIT_MERGE_KERNEL=cluster timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
timeout 120 python tools/host_overhead.py
timeout 120 python tools/timeline.py --dim 1000000 --workers 4
MARSIT_MERGE_KERNEL=cluster timeout 120 python tools/timeline.py --dim 1000000 --workers 4
timeout 120 python tools/timeline.py
