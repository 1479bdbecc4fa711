# Tile-height variants under the power cap (sustained 6000-step runs), and a
# parity subset on the TY=16 build.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
CAV_LIB=$PWD/build/ty16r7.so timeout 600 python -m pytest tests/test_gpu_run.py -m gpu -q -x -p no:cacheprovider -k "c1_full or stored or ragged" > gpurun_out/ty16_tests.log 2>&1; echo "ty16 tests exit $?"; tail -2 gpurun_out/ty16_tests.log
ROUNDS=2 STEPS=6000 bash scripts/gpu_ab.sh base=base ty16r7=build/ty16r7.so ty16r6=build/ty16r6.so > gpurun_out/ab_ty16.log 2>&1
cat gpurun_out/ab_ty16.log; cat gpurun_out/ab.txt
