cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build_native(defines=['MARSIT_CHECKED'], out='$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_checked.so')"
MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_checked.so STRESS_CONFIGS=80 timeout 1500 python tools/stress_determinism.py > gpurun_out/checked_stress.log 2>&1; echo stress_rc=$?; tail -3 gpurun_out/checked_stress.log
STRESS_SEED=7 STRESS_CONFIGS=60 timeout 900 python tools/stress_determinism.py > gpurun_out/stress_product.log 2>&1; echo stress_product_rc=$?; tail -3 gpurun_out/stress_product.log
