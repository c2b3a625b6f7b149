#!/bin/bash
# merge A/B on the box: GPU tests, merge-alone timings, per-step phases (debug build)
set -u
out=${1:-gpurun_out/merge_check.log}
timeout 900 python -m pytest tests -m gpu -x -q > ${out}.pytest 2>&1; echo "pytest rc=$?" >> ${out}.pytest
tail -2 ${out}.pytest > $out
for G in 8 4 2; do python tools/bench_merge_rank.py --ranks $G >> $out 2>&1; done
python tools/bench_merge_rank.py --ranks 8 --topo torus >> $out 2>&1
python tools/bench_merge.py >> $out 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > ${out}.bench 2>&1
python -c "import json; d=json.loads(open('${out}.bench').read().strip().splitlines()[-1]); print('bench us/step', d['ms_per_step']*1e3, d['phases_ms_per_step'], d['clocks'])" >> $out 2>&1
python -c "import __graft_entry__ as g; g.build_native(force=True, defines=['MARSIT_COOP_PROF'], out='/tmp/libprof.so')" && \
  MARSIT_SO=/tmp/libprof.so python tools/coop_prof.py >> $out 2>&1
