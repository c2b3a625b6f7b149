#!/bin/bash
# A/B: next round's coin precompute underneath the decode (0) or the extract (1)
run() {
  env $1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k,x in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for i in 1 2 3; do
  run MARSIT_COIN_PREFETCH_AT=0
  run MARSIT_COIN_PREFETCH_AT=1
done
