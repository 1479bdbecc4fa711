"""Diagnosis: long stored-ghost runs (fixed steps vs device-converged segments) against the oracle."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
from oracle.refbind import Oracle
from paper_2006_02602_b200 import capi

grid = (20, 16, 12)
N = int(os.environ.get("N", "12000"))
o = Oracle.run_case(capi.default_config(grid=grid, steps=N, check_every=10), collect_fields=True, collect_history=True)
oh = o["history"].view(np.uint64)
for sg in os.environ.get("GHOSTS", "0,1").split(","):
    os.environ["CAV_STORED_GHOSTS"] = sg
    for kind in os.environ.get("KINDS", "fixed,solve").split(","):
        if kind == "fixed":
            cfg = capi.default_config(grid=grid, steps=N, check_every=10)
        else:
            cfg = capi.default_config(grid=grid, steps=-1, conv_tol=1e-12, check_every=10)
            cfg.max_steps = N
        r = capi.run_case(cfg, collect_fields=True, collect_history=True)
        h = r.history.view(np.uint64)
        n = min(len(h), len(oh))
        bad = np.nonzero((h[:n] != oh[:n]).any(axis=1))[0]
        fbad = not np.array_equal(r.fields.view(np.uint64), o["fields"].view(np.uint64))
        print(f"ghosts={sg} {kind}: marched {r.steps_marched} rows {len(h)}/{len(oh)} "
              f"first bad row {bad[0] if len(bad) else None} (iteration {r.history_iter[bad[0]] if len(bad) else None}) "
              f"fields differ {fbad}", flush=True)
