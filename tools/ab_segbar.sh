#!/bin/bash
# A/B: per-segment barrier counters vs the grid barrier in the merge
for v in 0 1 0 1; do
  echo "SEG_BARRIER=$v"
  MARSIT_SEG_BARRIER=$v python tools/bench_merge.py 2>&1 | tail -1
  MARSIT_SEG_BARRIER=$v python tools/bench_merge_rank.py --ranks 2 2>&1 | tail -1
  MARSIT_SEG_BARRIER=$v python tools/bench_merge_rank.py --ranks 8 --topo torus 2>&1 | tail -1
  MARSIT_SEG_BARRIER=$v python tools/bench_merge_rank.py --ranks 8 2>&1 | tail -1
done
