cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
N=200000 GHOSTS=1 KINDS=solve,fixed timeout 900 python scripts/diag_solve.py > gpurun_out/diag_solve_long.log 2>&1; echo "diag_solve $?"; cat gpurun_out/diag_solve_long.log
timeout 600 python scripts/timing.py norms ranks > gpurun_out/timing_r02d.log 2>&1; echo "timing $?"; cat gpurun_out/timing_r02d.log
timeout 600 python bench.py > gpurun_out/bench_r02d.log 2>&1; echo "bench $?"; cat gpurun_out/bench_r02d.log
