# kernel variants bench + full GPU parity suite + ncu of the step kernel
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for K in tma tiled; do
  CAV_STEP_KERNEL=$K timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_$K.log 2>&1
  echo "bench $K exit $?"
done
timeout 300 python scripts/debug_overlap.py > gpurun_out/debug_overlap.log 2>&1; echo "dbg exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_tma python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tma.log 2>&1
echo "ncu exit $?"
