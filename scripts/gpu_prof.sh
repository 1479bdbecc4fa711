# bench + ncu full capture for TMA configs given as args
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for V in "$@"; do
  CAV_TMA_CFG=$V timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$V.log 2>&1; echo "bench v$V exit $?"
  CAV_TMA_CFG=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_v$V python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v$V.log 2>&1; echo "ncu v$V exit $?"
done
