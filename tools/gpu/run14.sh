cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_merge or large_segments or fused or anchors" 2>&1 | tail -3
for mk in grid cluster; do
for m in 0 1; do
export MARSIT_MERGE_KERNEL=$mk MARSIT_MERGE_MASKS=$m
echo "== $mk masks=$m"
echo -n "G8: "; MARSIT_MERGE_DEBUG=1 timeout 60 python tools/bench_merge_rank.py --ranks 8 2>&1 | grep -E "merge grid|per round" | tail -2 | tr '\n' ' '; echo
echo -n "C3: "; MARSIT_MERGE_DEBUG=1 timeout 60 python tools/bench_merge.py 2>&1 | grep -E "merge grid|stage 1|per round" | tail -2 | tr '\n' ' '; echo
echo -n "C4: "; timeout 60 python tools/bench_merge.py --dim 60200000 --topo torus --a 2 --b 4 2>&1 | tail -1
echo -n "C2: "; timeout 60 python tools/bench_merge.py --dim 61000000 2>&1 | tail -1
echo -n "C1: "; timeout 60 python tools/bench_merge.py --dim 1000000 --a 4 2>&1 | tail -1
done; done
