cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python scripts/debug_overlap2.py > gpurun_out/debug_overlap2.log 2>&1
echo "exit $?"
