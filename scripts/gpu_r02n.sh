# The whole GPU suite on the final build (re-run: the r02m box hung in cuInit before the first test).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,power.draw,clocks_event_reasons.active --format=csv
STALL=300 bash scripts/gpu_watchdog.sh n "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -3 gpurun_out/wd_n.log
