cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for C in 32 4; do
  CUDA_DEVICE_MAX_CONNECTIONS=$C timeout 200 python scripts/debug_overlap.py > gpurun_out/debug_conn$C.log 2>&1; echo "conn $C exit $?"
done
