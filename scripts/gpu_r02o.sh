cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_o.log 2>&1; echo "ranks fused $?"; cat gpurun_out/ranks_o.log
CAV_FUSED_HALO=0 ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_o_slab.log 2>&1; echo "ranks slab $?"; cat gpurun_out/ranks_o_slab.log
STALL=150 bash scripts/gpu_watchdog.sh o "python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_robustness.py tests/test_gpu_run.py tests/test_gpu_multiproc.py -m gpu -q -p no:cacheprovider"
tail -3 gpurun_out/wd_o.log
