cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STALL=150 bash scripts/gpu_watchdog.sh h "python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=5"
tail -8 gpurun_out/wd_h.log
ROUNDS=3 STEPS=1000 timeout 900 bash scripts/gpu_ab.sh head=build/head.so new=base > gpurun_out/ab_h.log 2>&1; tail -3 gpurun_out/ab_h.log
