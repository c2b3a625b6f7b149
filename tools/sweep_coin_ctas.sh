# Coin-prefetch residency vs. the decode it runs under (CUPTI timeline of the C3 step).
for c in 1 2 3 4 6; do echo "== MARSIT_COIN_CTAS=$c"; MARSIT_COIN_CTAS=$c python tools/timeline.py 2>&1 | tail -5; done
