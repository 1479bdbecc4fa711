# Final build (2x2 ghost kernel): smoke, driver-style and default bench lines, whole GPU suite, ncu launch list.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02r.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke_r02r.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20_r02r.log 2>&1; echo "bench20 exit $?"
timeout 900 python bench.py > gpurun_out/bench_r02r.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_r02r.log 2>&1; echo "bench ref exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02r.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_r02r.log 2>&1; echo "ncu launches exit $?"
STALL=300 bash scripts/gpu_watchdog.sh r "python -m pytest tests -m gpu -q -x -p no:cacheprovider"; tail -3 gpurun_out/wd_r.log
