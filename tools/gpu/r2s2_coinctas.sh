cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for r in 1 2; do for cc in 4 2 3 6; do echo -n "coin_ctas=$cc "; MARSIT_COIN_CTAS=$cc timeout 300 python tools/bench_configs.py --skip-c5 --configs c3 --iters 40 2>&1 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['sign_round_us'])"; done; done
