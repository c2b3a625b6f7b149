# compute-sanitizer evidence, ONE tool per gpurun call (B200_PROFILING.md):
#   bash tools/gpu/sanitize.sh <memcheck|racecheck|synccheck|initcheck>
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TOOL=${1:-memcheck}
CS=$(command -v compute-sanitizer || echo /usr/local/cuda/bin/compute-sanitizer)
# the plain run first: the sanitizer only runs on a program that exits 0
timeout 300 python tools/sanitize_round.py > gpurun_out/san_plain.log 2>&1 && \
SAN_DIM=4099 timeout 1500 $CS --tool $TOOL --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_round.py > gpurun_out/san_$TOOL.log 2>&1
echo "san_rc=$?"
tail -25 gpurun_out/san_$TOOL.log
