cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_share.log 2>&1; echo "ranks share $?"; cat gpurun_out/ranks_share.log
CAV_SHARE_SMS=0 ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_noshare.log 2>&1; echo "ranks noshare $?"; cat gpurun_out/ranks_noshare.log
timeout 300 python scripts/timing.py norms > gpurun_out/norms_new.log 2>&1; cat gpurun_out/norms_new.log
CAV_LIB=$PWD/build/old.so timeout 300 python scripts/timing.py norms > gpurun_out/norms_old.log 2>&1; cat gpurun_out/norms_old.log
cat > /tmp/normprof.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1)); b.initialize(); b.run(10)
b.run(6, check_every=1, want_norms=True); b.close()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/norm_launches.csv python /tmp/normprof.py > /dev/null 2>&1; echo "ncu $?"
grep -o '"k_[a-z_]*[^"]*","[^"]*","gpu__time_duration.sum","[^"]*","[0-9.]*"' gpurun_out/norm_launches.csv | tail -20
