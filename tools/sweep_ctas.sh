for cfg in "3 2 4 1" "2 2 4 1" "3 2 4 0" "3 2 8 0"; do
  set -- $cfg
  echo "== extract=$1 decode=$2 coins=$3 nopipe=$4"
  if [ "$4" = "1" ]; then export MARSIT_NO_PIPELINE=1; else unset MARSIT_NO_PIPELINE; fi
  MARSIT_EXTRACT_CTAS=$1 MARSIT_DECODE_CTAS=$2 MARSIT_COIN_CTAS=$3 timeout 200 python tools/timeline.py 2>/dev/null | tail -20
done
