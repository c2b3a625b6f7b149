cd $GRAFT_REPO_ROOT
for cc in 1 2 4; do for dc in 2 3; do
  echo -n "coin_ctas=$cc decode_ctas=$dc: "
  MARSIT_COIN_CTAS=$cc MARSIT_DECODE_CTAS=$dc python bench.py --no-cpu-baseline --steps 30 --min-busy-s 0.5 --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']
print(round(d['ms_per_step']*1e3,1), 'us; decode', round(p['decode_comp']*1e3,1), 'coins', round(p.get('coins',0)*1e3,1), 'merge', round(p['merge']*1e3,1), 'extract', round(p['sign_extract']*1e3,1), d['clocks']['sm_mhz'])"
done; done
echo -n "prefetch at extract: "; MARSIT_COIN_PREFETCH_AT=1 python bench.py --no-cpu-baseline --steps 30 --min-busy-s 0.5 --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']
print(round(d['ms_per_step']*1e3,1), 'us; decode', round(p['decode_comp']*1e3,1), 'coins', round(p.get('coins',0)*1e3,1), 'extract', round(p['sign_extract']*1e3,1))"
