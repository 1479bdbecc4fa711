cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ROUNDS=3 STEPS=1000 timeout 900 bash scripts/gpu_ab.sh head=build/head.so new=base > gpurun_out/ab_i.log 2>&1; tail -3 gpurun_out/ab_i.log
STALL=150 bash scripts/gpu_watchdog.sh i "python -m pytest tests/test_gpu_run.py tests/test_gpu_fuzz.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider -k 'stored or ghost or fuzz or c1_full or solve or linf'"
tail -3 gpurun_out/wd_i.log
