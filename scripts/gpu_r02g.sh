cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ROUNDS=2 STEPS=1000 timeout 900 bash scripts/gpu_ab.sh old=build/old.so new=base > gpurun_out/ab_g.log 2>&1; tail -3 gpurun_out/ab_g.log
ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_g.log 2>&1; echo "ranks $?"; cat gpurun_out/ranks_g.log
STALL=120 bash scripts/gpu_watchdog.sh g "python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_robustness.py tests/test_gpu_multiproc.py -m gpu -q -x -p no:cacheprovider"
tail -3 gpurun_out/wd_g.log
