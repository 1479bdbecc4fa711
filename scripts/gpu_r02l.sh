cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
echo "== current, slab path"; CAV_FUSED_HALO=0 OV=1 STEPS=50 REPS=10 timeout 600 python scripts/diag_c2.py | grep -c " 0 mismatches"
echo "== head.so"; CAV_LIB=$PWD/build/head.so OV=1 STEPS=50 REPS=10 timeout 600 python scripts/diag_c2.py | grep -c " 0 mismatches"
echo "== current, fused"; OV=1 STEPS=50 REPS=10 timeout 600 python scripts/diag_c2.py | grep -c " 0 mismatches"
echo "== current, fused 2d np4 512"; GRID=256,256,512 NP=4 MODE=2d OV=1 STEPS=30 REPS=5 timeout 600 python scripts/diag_c2.py | grep -c " 0 mismatches"
