set -x
ls -la /usr/local/cuda/compute-sanitizer 2>&1 | head -3; which compute-sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest1.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest1.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
