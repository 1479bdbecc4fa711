# Norm helper warps (stored-ghost norm iterations without the residual scratch round trip):
# timing with/without (CAV_NORM_HELPER), then the GPU suite.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for h in 1 0 1; do
  echo "== CAV_NORM_HELPER=$h"; CAV_NORM_HELPER=$h timeout 180 python scripts/timing.py norms; echo "exit $?"
done > gpurun_out/norm_helper_ab.log 2>&1
cat gpurun_out/norm_helper_ab.log
STALL=150 bash scripts/gpu_watchdog.sh j "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -5 gpurun_out/wd_j.log
