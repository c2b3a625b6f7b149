cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_merge or large_segments or fused" 2>&1 | tail -2
for pf in 0 1; do
export MARSIT_MERGE_PREFETCH=$pf
echo "== prefetch=$pf"
echo -n "G8: "; timeout 60 python tools/bench_merge_rank.py --ranks 8 2>&1 | tail -1
echo -n "G8 torus: "; timeout 60 python tools/bench_merge_rank.py --ranks 8 --topo torus 2>&1 | tail -1
echo -n "G2: "; timeout 60 python tools/bench_merge_rank.py --ranks 2 2>&1 | tail -1
echo -n "C3: "; timeout 60 python tools/bench_merge.py 2>&1 | tail -1
echo -n "C4: "; timeout 60 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
echo -n "C2: "; timeout 60 python tools/bench_merge.py --dim 61000000 2>&1 | tail -1
done
