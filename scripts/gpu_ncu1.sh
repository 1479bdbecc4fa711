# one ncu --set full capture of the step kernel (variant $1, tag $2)
cd $GRAFT_REPO_ROOT
CAV_TMA_CFG=${1:-0} timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_$2 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$2.log 2>&1; echo "ncu exit $?"
