cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python scripts/timing.py norms > gpurun_out/norms_r.log 2>&1; echo "norms"; cat gpurun_out/norms_r.log
CAV_LIB=$PWD/build/base1.so timeout 300 python scripts/timing.py norms > gpurun_out/norms_r0.log 2>&1; echo "norms base"; cat gpurun_out/norms_r0.log
STALL=150 bash scripts/gpu_watchdog.sh r "python -m pytest tests/test_gpu_run.py tests/test_gpu_robustness.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k 'stored or ghost or solve or linf or c1_256 or 512cube or fuzz'"
tail -3 gpurun_out/wd_r.log
