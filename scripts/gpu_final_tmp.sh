cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for r in 1 2; do
  STALL=150 bash scripts/gpu_watchdog.sh z$r "python -m pytest tests -m gpu -q -p no:cacheprovider"
  tail -1 gpurun_out/wd_z$r.log
done
STALL=200 bash scripts/gpu_watchdog.sh zf "python scripts/fuzz_wide.py 400 600"; tail -2 gpurun_out/wd_zf.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
cat > /tmp/normprof.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1)); b.initialize(); b.run(10)
b.run(6, check_every=1, want_norms=True); b.close()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/norm_launches_z.csv python /tmp/normprof.py > /dev/null 2>&1; echo "ncu $?"
