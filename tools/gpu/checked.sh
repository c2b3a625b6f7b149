# Checked build (jitter at every merge barrier + device index bounds) through
# the GPU parity suites and the randomised determinism stress.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
export MARSIT_SO=$GRAFT_REPO_ROOT/paper_2204_06787_b200/libmarsit_b200_checked.so
# (re)build the checked variant of the library when a source is newer
python -c "import __graft_entry__ as g; g.build_native(defines=['MARSIT_CHECKED'], out='$MARSIT_SO')"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_multirank_emulated.py tests/test_gpu_metrics.py tests/test_gpu_driver.py tests/test_gpu_failure.py -x -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo checked_pytest_rc=$?; tail -4 gpurun_out/checked_pytest.log
timeout 1200 python tools/stress_determinism.py > gpurun_out/checked_stress.log 2>&1; echo stress_rc=$?; tail -5 gpurun_out/checked_stress.log
unset MARSIT_SO
STRESS_SEED=7 timeout 900 python tools/stress_determinism.py > gpurun_out/stress_product.log 2>&1; echo stress_product_rc=$?; tail -3 gpurun_out/stress_product.log
