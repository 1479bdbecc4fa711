# GPU parity suite + smoke (+ optional bench), results in gpurun_out/
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
if [ "$1" = "bench" ]; then
  timeout 300 python bench.py --steps 2000 --warmup 20 --cpu-seconds 10 > gpurun_out/bench.log 2>&1
  echo "bench exit $?"
fi
