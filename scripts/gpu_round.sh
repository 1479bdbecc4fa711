# Round evidence: full bench line, ncu launch list of the same command, one
# ncu --set full capture of the step kernel, GPU tests and smoke.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?"
timeout 300 python bench.py --gpus 2 --steps 200 --warmup 5 --no-e2e > gpurun_out/bench2_$TAG.log 2>&1; echo "bench2 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full exit $?"
if [ "$2" != "notests" ]; then
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?"
