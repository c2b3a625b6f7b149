cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in A B A B; do
  if [ $v = A ]; then export MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_A.so; else unset MARSIT_SO; fi
  echo -n "$v: "; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control base -k regex:coins_kernel -s 5 -c 3 python bench.py --steps 3 --warmup 3 --min-busy-s 0 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "duration" | awk '{printf "%s ", $3}'; echo
done
