cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_coins.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "coin or fused or spread or golden or c3" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:coins_kernel -s 5 -c 2 python bench.py --steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "duration|pipe_" 
timeout 300 python tools/bench_configs.py --skip-c5 --configs c3,c4 --iters 40 2>&1 | cut -c1-200 | head -6
timeout 600 python bench.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['frac'], d['phases_ms_per_step'], d['clocks'])"
