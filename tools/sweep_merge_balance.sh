# Merge tiling sweep (merge alone): words per thread x CTAs per SM.
for WK in "0 0" "4 0" "8 0" "12 0" "16 0" "12 2" "16 2"; do set -- $WK
  echo -n "C3 wpt=$1 k=$2: "; MARSIT_MERGE_WPT=$1 MARSIT_MERGE_BALANCE=$2 python tools/bench_merge.py 2>&1 | tail -1
done
for G in 8 4 2; do for WK in "0 0" "1 0" "2 0" "4 0" "8 0" "12 0" "16 0" "4 1" "8 1" "16 1" "8 2" "12 2"; do set -- $WK
  echo -n "G=$G wpt=$1 k=$2: "; MARSIT_MERGE_WPT=$1 MARSIT_MERGE_BALANCE=$2 python tools/bench_merge_rank.py --ranks $G 2>&1 | tail -1
done; done
for WK in "0 0" "2 0" "4 0" "8 0"; do set -- $WK
  echo -n "torus G=8 wpt=$1 k=$2: "; MARSIT_MERGE_WPT=$1 MARSIT_MERGE_BALANCE=$2 python tools/bench_merge_rank.py --topo torus 2>&1 | tail -1
done
