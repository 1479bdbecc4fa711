# Upper bound of the last CTA's centre-cell fold on the iteration time: a probe build without it (wrong pcs, timing only).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ROUNDS=3 STEPS=100 bash scripts/gpu_ab.sh base=base nocenter=build/nocenter.so > gpurun_out/ab_r02s.log 2>&1
grep AB gpurun_out/ab_r02s.log
