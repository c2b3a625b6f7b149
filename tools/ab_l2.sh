#!/bin/bash
# A/B of the K1/K4 task-order L2 reuse: bench step time per setting
run() {
  env $1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k,x in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for i in 1 2; do
  run MARSIT_L2_REUSE=0
  run MARSIT_L2_REUSE=1
done
