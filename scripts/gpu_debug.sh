cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 120 python scripts/debug_exchange.py > gpurun_out/debug_exchange.log 2>&1
echo "debug exit $?"
bash scripts/gpu_quick.sh
