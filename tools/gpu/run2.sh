# GPU session 2: failure tests, cluster-merge parity, merge timings
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 180 python -m pytest tests/test_gpu_failure.py -x -q > gpurun_out/t_failure.log 2>&1; echo failure_rc=$? ; tail -15 gpurun_out/t_failure.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_metrics.py -x -q > gpurun_out/t_parity.log 2>&1; echo parity_rc=$?; tail -15 gpurun_out/t_parity.log
timeout 600 python -m pytest tests/test_gpu_multirank_emulated.py tests/test_gpu_driver.py tests/test_gpu_ssdm.py tests/test_gpu_p2p_ipc.py -x -q > gpurun_out/t_multi.log 2>&1; echo multi_rc=$?; tail -15 gpurun_out/t_multi.log
for cs in 0; do
 timeout 120 python tools/bench_merge.py 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 61000000 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
 for G in 8 4 2; do timeout 120 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1; done
 timeout 120 python tools/bench_merge_rank.py --ranks 8 --topo torus 2>&1 | tail -1
done
echo "--- coop (round-1 kernel) ---"
export MARSIT_MERGE_COOP=1
 timeout 120 python tools/bench_merge.py 2>&1 | tail -1
 timeout 120 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
 for G in 8 2; do timeout 120 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1; done
unset MARSIT_MERGE_COOP
timeout 300 python tools/bench_configs.py --skip-c5 --iters 20 > gpurun_out/configs2.jsonl 2>&1; echo configs_rc=$?; cat gpurun_out/configs2.jsonl | head -30
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench2.json 2>gpurun_out/bench2.err; echo bench_rc=$?; cat gpurun_out/bench2.json
