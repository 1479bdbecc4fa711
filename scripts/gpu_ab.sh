# Interleaved A/B timing of alternate library builds (CAV_LIB): each arg is
# NAME=path/to/lib.so ("base" = the in-tree build). ROUNDS x STEPS per run.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
ROUNDS=${ROUNDS:-3}
STEPS=${STEPS:-600}
: > gpurun_out/ab.txt
for r in $(seq $ROUNDS); do
  for A in "$@"; do
    NAME=${A%%=*}; LIBP=${A#*=}
    if [ "$LIBP" = "base" ]; then unset CAV_LIB; else export CAV_LIB=$PWD/$LIBP; fi
    timeout 300 python bench.py --steps $STEPS --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ab_run.log 2>&1
    python - "$NAME" >> gpurun_out/ab.txt <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/ab_run.log").read().strip().splitlines()[-1])
    print(sys.argv[1], d["roofline"]["kernel_ms"], d["value"])
except Exception as e: print(sys.argv[1], "fail", 0)
PY
  done
done
unset CAV_LIB
python - <<'PY'
from collections import defaultdict
t=defaultdict(list)
for line in open("gpurun_out/ab.txt"):
    n,ms,v=line.split(); 
    if ms!="fail": t[n].append(float(ms))
for n,v in t.items(): print(f"AB {n:12s} mean {sum(v)/len(v):.4f} ms  min {min(v):.4f}  n={len(v)}  -> {16777216/ (sum(v)/len(v)) / 1e3:.0f} MCUPS")
PY
