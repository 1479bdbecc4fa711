cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STALL=120 bash scripts/gpu_watchdog.sh f "python -m pytest tests -m gpu -q -x -p no:cacheprovider -k 'not c1_256cube and not 512cube'"
tail -4 gpurun_out/wd_f.log
ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_f.log 2>&1; echo "ranks $?"; cat gpurun_out/ranks_f.log
