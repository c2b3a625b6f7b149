# Merge tiling sweep: words per thread (WPT) x CTAs per SM (MARSIT_MERGE_BALANCE).
for G in 8 4 2; do for W in 0 1 2 4 8; do
  echo -n "G=$G wpt=$W: "; MARSIT_MERGE_WPT=$W python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1
done; done
for W in 0 2 4 8; do echo -n "torus G=8 wpt=$W: "; MARSIT_MERGE_WPT=$W python tools/bench_merge_rank.py --topo torus 2>&1 | tail -1; done
for W in 0 4 8; do echo -n "C3 1-GPU wpt=$W: "; MARSIT_MERGE_WPT=$W python tools/bench_merge.py 2>&1 | tail -1; done
