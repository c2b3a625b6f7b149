cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for cs in 0 128 112 96 80 64; do echo -n "G8 cs=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1; done
for cs in 0 112 96 80 64 48; do echo -n "G8torus cs=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge_rank.py --ranks 8 --topo torus --iters 100 2>&1 | tail -1; done
for cs in 0 64 56 48 40 32; do echo -n "G4 cs=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge_rank.py --ranks 4 --iters 100 2>&1 | tail -1; done
for cs in 0 32 28 24 20; do echo -n "G2 cs=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge_rank.py --ranks 2 --iters 100 2>&1 | tail -1; done
for cs in 0 16 14; do echo -n "C3 cs=$cs: "; MARSIT_MERGE_CSIZE=$cs timeout 60 python tools/bench_merge.py --iters 100 2>&1 | tail -1; done
