for i in 1 2 3; do for e in 3 4; do
  echo -n "E=$e: "; MARSIT_EXTRACT_CTAS=$e python tools/timeline.py 2>&1 | grep -E "step span|StreamParams" | head -2 | tr '\n' ' ' | sed -E 's/ +/ /g' | cut -c1-160; echo
done; done
