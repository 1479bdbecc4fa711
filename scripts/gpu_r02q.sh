# y/z ghost kernel variants: two rows per thread with the stop check after the loads (CAV_GHOST_PAIRS=2) vs pairs (1) vs single (0).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
CAV_GHOST_PAIRS=2 timeout 900 python -m pytest tests/test_gpu_run.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/g4_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/g4_tests.log
ROUNDS=3 STEPS=100 bash scripts/gpu_ab.sh pairs=base rows2=base+CAV_GHOST_PAIRS=2 single=base+CAV_GHOST_PAIRS=0 > gpurun_out/ab_r02q_burst.log 2>&1
for v in 2 1; do CAV_GHOST_PAIRS=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ghosts -c 10 --csv --log-file gpurun_out/g4_ncu_$v.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $v exit $?"; done
grep AB gpurun_out/ab_r02q_burst.log
