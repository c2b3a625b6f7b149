cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for pf in 0 1 2 3; do
export MARSIT_MERGE_PREFETCH=$pf
echo -n "pf=$pf G8: "; timeout 60 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
echo -n "pf=$pf C3: "; timeout 60 python tools/bench_merge.py --iters 100 2>&1 | tail -1
echo -n "pf=$pf C4: "; timeout 60 python tools/bench_merge.py --iters 50 --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
done; done
