# TMA step kernel configuration sweep (bench at 256^3) + quick parity
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for V in 0 1 2 3; do
  CAV_TMA_CFG=$V timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$V.log 2>&1
  echo "bench v$V exit $?"
done
timeout 600 python -m pytest tests/test_gpu_run.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "serial or parallel_c0 or block or fused" > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?"
