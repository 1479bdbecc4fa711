# Re-entry check of HEAD on a fresh box: default bench line, then the whole GPU suite.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r02g.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_r02g.log | cut -c1-400
STALL=150 bash scripts/gpu_watchdog.sh g "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -3 gpurun_out/wd_g.log
