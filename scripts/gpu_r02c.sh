cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STALL=120 bash scripts/gpu_watchdog.sh rb "python -m pytest tests/test_gpu_robustness.py tests/test_gpu_run.py -m gpu -q -p no:cacheprovider -k 'robustness or ragged or solve'"
tail -5 gpurun_out/wd_rb.log
timeout 600 python scripts/diag_solve.py > gpurun_out/diag_solve.log 2>&1; echo "diag_solve $?"; cat gpurun_out/diag_solve.log
ROUNDS=2 STEPS=1000 timeout 900 bash scripts/gpu_ab.sh p3=base+CAV_L2_PROMO=3 p0=base+CAV_L2_PROMO=0 p1=base+CAV_L2_PROMO=1 p2=base+CAV_L2_PROMO=2 > gpurun_out/ab_promo.log 2>&1; tail -5 gpurun_out/ab_promo.log
