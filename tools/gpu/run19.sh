cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_merge or large_segments" 2>&1 | tail -2
for rep in 1 2; do
for pf in 0 1; do
export MARSIT_MERGE_COIN_PF=$pf
echo -n "cpf=$pf G8: "; timeout 60 python tools/bench_merge_rank.py --ranks 8 --iters 100 2>&1 | tail -1
echo -n "cpf=$pf C3: "; timeout 60 python tools/bench_merge.py --iters 100 2>&1 | tail -1
echo -n "cpf=$pf C4: "; timeout 60 python tools/bench_merge.py --iters 50 --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
done; done
