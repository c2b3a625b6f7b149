cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
export MARSIT_MERGE_KERNEL=grid
for cs in 0 96 64 48 32 16; do echo -n "G8 csize=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge_rank.py --ranks 8 2>&1 | tail -1; done
for cs in 0 12 9 6; do echo -n "C3 csize=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge.py 2>&1 | tail -1; done
for cs in 0 12; do echo -n "C4 csize=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1; done
echo -n "C1: "; timeout 60 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
