cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python scripts/timing.py norms > gpurun_out/norms_q.log 2>&1; echo "norms runs"; cat gpurun_out/norms_q.log
CAV_NORM_RUNS=0 timeout 300 python scripts/timing.py norms > gpurun_out/norms_q0.log 2>&1; echo "norms scratch"; cat gpurun_out/norms_q0.log
STALL=150 bash scripts/gpu_watchdog.sh q "python -m pytest tests/test_gpu_run.py tests/test_gpu_robustness.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k 'stored or ghost or solve or linf or c1_256 or 512cube or fuzz'"
tail -3 gpurun_out/wd_q.log
