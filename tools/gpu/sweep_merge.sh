cd $GRAFT_REPO_ROOT
for w in 8 12 16; do for k in 0 1 2 3; do echo -n "C3 wpt=$w k=$k: "; MARSIT_MERGE_WPT=$w MARSIT_MERGE_BALANCE=$k timeout 60 python tools/bench_merge.py 2>&1 | tail -1; done; done
for w in 1 2 4; do for k in 0 1 2; do echo -n "G8 wpt=$w k=$k: "; MARSIT_MERGE_WPT=$w MARSIT_MERGE_BALANCE=$k timeout 60 python tools/bench_merge_rank.py --ranks 8 2>&1 | tail -1; done; done
