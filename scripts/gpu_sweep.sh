# comm-priority hang check + TMA step kernel configuration sweep
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 400 python scripts/debug_overlap.py > gpurun_out/debug_overlap.log 2>&1; echo "dbg exit $?"
for V in 0 1 2 3; do
  CAV_TMA_CFG=$V timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$V.log 2>&1
  echo "bench v$V exit $?"
done
