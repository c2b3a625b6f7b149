cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
MARSIT_MERGE_DEBUG=1 timeout 120 python tools/bench_merge.py 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_multirank_emulated.py -x -q > gpurun_out/t_parity4.log 2>&1; echo parity_rc=$?; tail -5 gpurun_out/t_parity4.log
 timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
 for G in 8 2; do timeout 120 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1; done
 timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus 2>&1 | tail -1
 for cs in 8 10 12 14; do echo cs=$cs; MARSIT_MERGE_CSIZE=$cs timeout 120 python tools/bench_merge.py 2>&1 | tail -1; done
