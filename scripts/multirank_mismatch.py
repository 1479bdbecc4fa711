"""Multi-rank GPU runs vs the one-rank GPU run of the same case, repeated
(REPS) to catch rare races: prints how many cells differ and where (per
variable k/j/i ranges). Env: GRID, NP, MODE, STEPS, REPS, OV, HIST.
Round 2 used it to find a slab-path unpack that skipped a stale flag."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
from paper_2006_02602_b200 import capi

grid = tuple(int(x) for x in os.environ.get("GRID", "256,256,256").split(","))
np_ = int(os.environ.get("NP", "8"))
mode = os.environ.get("MODE", "1d-i")
_want = {}
for steps in [int(x) for x in os.environ.get("STEPS", "2,5,50").split(",")] * int(os.environ.get("REPS", "1")):
    hist = os.environ.get("HIST", "1") == "1"
    if steps not in _want:
        _want[steps] = capi.run_case(capi.default_config(grid=grid, steps=steps, check_every=5), collect_fields=True,
                                     collect_history=hist)
    want = _want[steps]
    for ov in [int(x) for x in os.environ.get("OV", "1,0").split(",")]:
        got = capi.run_case(capi.default_config(grid=grid, steps=steps, check_every=5, np=np_, mode=mode,
                                                strategy="v3", overlap=ov), collect_fields=True,
                            collect_history=hist)
        a, b = got.fields.view(np.uint64), want.fields.view(np.uint64)
        bad = np.argwhere(a != b)
        msg = f"steps={steps} overlap={ov}: {len(bad)} mismatches"
        if len(bad):
            for v in range(5):
                bv = bad[bad[:, 0] == v]
                if len(bv):
                    msg += f"\n   var {v}: {len(bv)}  k {bv[:,1].min()}..{bv[:,1].max()}  j {bv[:,2].min()}..{bv[:,2].max()}  i {bv[:,3].min()}..{bv[:,3].max()}  i-values {sorted(set(bv[:,3].tolist()))[:12]}"
        print(msg, flush=True)
