cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python scripts/debug_overlap.py > gpurun_out/debug_overlap.log 2>&1; echo "dbg exit $?"
timeout 300 python bench.py --steps 2000 --warmup 20 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
