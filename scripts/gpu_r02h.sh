# L2 cache hints on the TMA tile loads and k-chunk lengths, sustained (2000 steps, power cap) and burst (100 steps).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ROUNDS=2 STEPS=2000 bash scripts/gpu_ab.sh base=base hint1=build/hint1.so hint2=build/hint2.so c32=base+CAV_TMA_CHUNK=32 c64=base+CAV_TMA_CHUNK=64 c96=base+CAV_TMA_CHUNK=96 > gpurun_out/ab_r02h_sustained.log 2>&1
cp gpurun_out/ab.txt gpurun_out/ab_r02h_sustained_raw.txt
ROUNDS=2 STEPS=100 bash scripts/gpu_ab.sh base=base hint1=build/hint1.so hint2=build/hint2.so c64=base+CAV_TMA_CHUNK=64 > gpurun_out/ab_r02h_burst.log 2>&1
cat gpurun_out/ab_r02h_sustained.log gpurun_out/ab_r02h_burst.log
