# Programmatic dependent launch (CAV_PDL=1) of the plain step and the y/z ghost kernel: sanity, parity subset, A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
CAV_PDL=1 timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl_sanity.log 2>&1; echo "sanity exit $?"; tail -1 gpurun_out/pdl_sanity.log | cut -c1-160
CAV_PDL=1 timeout 900 python -m pytest tests/test_gpu_run.py tests/test_gpu_fuzz.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pdl_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/pdl_tests.log
ROUNDS=3 STEPS=100 bash scripts/gpu_ab.sh base=base pdl=base+CAV_PDL=1 > gpurun_out/ab_r02p_burst.log 2>&1
ROUNDS=2 STEPS=2000 bash scripts/gpu_ab.sh base=base pdl=base+CAV_PDL=1 > gpurun_out/ab_r02p_sustained.log 2>&1
grep AB gpurun_out/ab_r02p_burst.log gpurun_out/ab_r02p_sustained.log
