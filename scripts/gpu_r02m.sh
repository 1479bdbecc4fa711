# Final-build check on a fresh B200: smoke, default bench line, driver-style short bench, the whole GPU suite.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02m.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke_r02m.log
timeout 900 python bench.py > gpurun_out/bench_r02m.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20_r02m.log 2>&1; echo "bench20 exit $?"
STALL=150 bash scripts/gpu_watchdog.sh m "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -3 gpurun_out/wd_m.log
