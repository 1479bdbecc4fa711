cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python scripts/debug_overlap.py > gpurun_out/debug_overlap.log 2>&1; echo "dbg exit $?"
