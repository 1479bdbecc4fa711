# k_norm_runs load-batch depth under ncu: duration, DRAM bytes, issue activity
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
cat > /tmp/normprof.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1))
b.initialize()
b.run(4)
secs, chk = b.run(4, check_every=1, want_norms=True)
print("ok", len(chk))
b.close()
PY
for a in 1 8; do
CAV_NORM_AHEAD=$a timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/norms_ncu_$a.csv python /tmp/normprof.py > gpurun_out/ncu_norms_$a.log 2>&1; echo "ncu $a exit $?"
done
