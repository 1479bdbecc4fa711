# Wide fuzz on the final build (new seeds 600..900), three exchange/ghost variants per draw, against the oracle.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STALL=300 bash scripts/gpu_watchdog.sh o "timeout 1500 python scripts/fuzz_wide.py 600 900"; tail -3 gpurun_out/wd_o.log
