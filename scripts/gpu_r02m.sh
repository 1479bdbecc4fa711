cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
echo "== current, slab path"; CAV_FUSED_HALO=0 OV=1 STEPS=50 REPS=40 timeout 900 python scripts/diag_c2.py | grep -v " 0 mismatches" | head -8
echo "== head.so"; CAV_LIB=$PWD/build/head.so OV=1 STEPS=50 REPS=40 timeout 900 python scripts/diag_c2.py | grep -v " 0 mismatches" | head -8
echo "== current, fused"; OV=1 STEPS=50 REPS=40 timeout 900 python scripts/diag_c2.py | grep -v " 0 mismatches" | head -8
echo done
