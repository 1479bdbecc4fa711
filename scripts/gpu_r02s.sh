cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
echo "graphs"; timeout 300 python scripts/timing.py runs solve
echo "no graphs"; CAV_GRAPHS=0 timeout 300 python scripts/timing.py runs solve
STALL=150 bash scripts/gpu_watchdog.sh t "python -m pytest tests -m gpu -q -x -p no:cacheprovider -k 'not c1_256cube and not 512cube'"
tail -3 gpurun_out/wd_t.log
