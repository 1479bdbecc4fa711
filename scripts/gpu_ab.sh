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
    # optional environment for this variant: LIB+VAR=VALUE
    VENV=""; case "$LIBP" in *+*) VENV=${LIBP#*+}; LIBP=${LIBP%%+*};; esac
    if [ "$LIBP" = "base" ]; then unset CAV_LIB; else export CAV_LIB=$PWD/$LIBP; fi
    env $VENV timeout 300 python bench.py --steps $STEPS --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ab_run.log 2>&1
    python - "$NAME" >> gpurun_out/ab.txt <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/ab_run.log").read().strip().splitlines()[-1])
    print(sys.argv[1], d["roofline"]["kernel_ms"], d["value"], d["ms_per_step"])
except Exception as e: print(sys.argv[1], "fail", 0)
PY
  done
done
unset CAV_LIB
python - <<'PY'
from collections import defaultdict
t=defaultdict(list)
for line in open("gpurun_out/ab.txt"):
    f=line.split()
    if f[1]!="fail": t[f[0]].append((float(f[1]), float(f[3])))
for n,v in t.items():
    k=sum(x[0] for x in v)/len(v); s=sum(x[1] for x in v)/len(v)
    print(f"AB {n:12s} kernel {k:.4f} ms  step {s:.4f} ms  n={len(v)}  -> step {16777216/s/1e3:.0f} MCUPS")
PY
