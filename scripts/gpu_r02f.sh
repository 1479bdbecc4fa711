# HEAD check: default bench line, then the whole GPU suite.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r02f.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_r02f.log | cut -c1-400
STALL=150 bash scripts/gpu_watchdog.sh f "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -3 gpurun_out/wd_f.log
