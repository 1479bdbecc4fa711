# correctness (smoke) + bench for every TMA step variant given as args (CAV_TMA_CFG)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for V in "$@"; do
  CAV_TMA_CFG=$V timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v$V.log 2>&1; echo "smoke v$V exit $?"
  CAV_TMA_CFG=$V timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$V.log 2>&1; echo "bench v$V exit $?"
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_v$V.log").read().strip().splitlines()[-1])
    print("v$V", round(d["value"]), "MCUPS frac", round(d["roofline"]["frac"],3), "kernel_ms", round(d["roofline"]["kernel_ms"],4), d["clocks"])
except Exception as e: print("v$V parse fail", e)
PY
done
