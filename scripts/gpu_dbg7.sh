cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 200 python scripts/debug_overlap.py > gpurun_out/debug_1stream.log 2>&1; echo "1stream exit $?"
CAV_OVERLAP_STREAMS=2 timeout 200 python scripts/debug_overlap.py > gpurun_out/debug_2stream.log 2>&1; echo "2stream exit $?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
