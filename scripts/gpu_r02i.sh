# setmaxnreg (issuer warpgroup at 24 registers, consumers at 104) and the
# 16-byte pair-load probe: quick sanity run, then sustained and burst A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in smr104 smr104pair; do
  CAV_LIB=$PWD/build/$v.so timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sanity_$v.log 2>&1
  echo "sanity $v exit $?"; tail -1 gpurun_out/sanity_$v.log | cut -c1-200
done
CAV_LIB=$PWD/build/smr104.so timeout 600 python -m pytest tests/test_gpu_run.py -m gpu -q -x -p no:cacheprovider -k "c1_full or stored or ragged" > gpurun_out/smr104_tests.log 2>&1; echo "smr104 tests exit $?"; tail -2 gpurun_out/smr104_tests.log
ROUNDS=2 STEPS=2000 bash scripts/gpu_ab.sh base=base smr104=build/smr104.so pair=build/pairprobe.so smr104pair=build/smr104pair.so > gpurun_out/ab_r02i_sustained.log 2>&1
ROUNDS=2 STEPS=100 bash scripts/gpu_ab.sh base=base smr104=build/smr104.so pair=build/pairprobe.so smr104pair=build/smr104pair.so > gpurun_out/ab_r02i_burst.log 2>&1
cat gpurun_out/ab_r02i_sustained.log gpurun_out/ab_r02i_burst.log
