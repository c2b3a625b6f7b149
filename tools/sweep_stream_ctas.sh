# Residency of the streaming kernels (CUPTI timeline of the C3 step).
for e in 2 3 4; do for d in 2 3; do
  echo "== EXTRACT_CTAS=$e DECODE_CTAS=$d"
  MARSIT_EXTRACT_CTAS=$e MARSIT_DECODE_CTAS=$d python tools/timeline.py 2>&1 | grep -E "StreamParams|step span" | sed -E 's/ +/ /g' | cut -c1-120
done; done
