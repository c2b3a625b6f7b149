cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for cs in 1 2 4 8 16; do echo "csize $cs"; MARSIT_MERGE_KERNEL=cluster MARSIT_MERGE_CSIZE=$cs timeout 120 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1; done
for cs in 4 8 16; do echo "G=8 csize $cs"; MARSIT_MERGE_KERNEL=cluster MARSIT_MERGE_CSIZE=$cs timeout 120 python tools/bench_merge_rank.py --ranks 8 2>&1 | tail -1; done
timeout 120 python tools/timeline.py --dim 1000000 --workers 4 2>&1 | grep -v -i warn
MARSIT_FUSED=0 timeout 120 python tools/timeline.py --dim 1000000 --workers 4 2>&1 | grep -v -i warn
MARSIT_FUSED=0 MARSIT_MERGE_KERNEL=cluster MARSIT_MERGE_CSIZE=1 timeout 120 python tools/timeline.py --dim 1000000 --workers 4 2>&1 | grep -v -i warn
