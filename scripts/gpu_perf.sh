# bench + full GPU suite + ncu (launch list and full capture of the step kernel)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python bench.py --steps 2000 --warmup 20 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_tma python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tma.log 2>&1; echo "ncu2 exit $?"
