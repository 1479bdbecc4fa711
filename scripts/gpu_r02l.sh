# Paired-column y/z wall-ghost kernel (k_ghosts_yz2): parity subset, A/B against k_ghosts_yz, launch durations.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_run.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ghost2_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/ghost2_tests.log
ROUNDS=3 STEPS=100 bash scripts/gpu_ab.sh pairs=base single=base+CAV_GHOST_PAIRS=0 > gpurun_out/ab_r02l_burst.log 2>&1
ROUNDS=2 STEPS=2000 bash scripts/gpu_ab.sh pairs=base single=base+CAV_GHOST_PAIRS=0 > gpurun_out/ab_r02l_sustained.log 2>&1
for v in 1 0; do CAV_GHOST_PAIRS=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ghosts -c 10 --csv --log-file gpurun_out/ghosts_ncu_$v.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $v exit $?"; done
cat gpurun_out/ab_r02l_burst.log gpurun_out/ab_r02l_sustained.log | grep AB
