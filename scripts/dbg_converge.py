# C0 to convergence (cavity solve's default mode) on the GPU: iterations and wall time.
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
capi.run_case(capi.default_config(grid=(16, 16, 16), steps=20))  # CUDA context + module load
for grid in ((32, 32, 32), (64, 64, 64)):
    cfg = capi.default_config(grid=grid, steps=-1)
    t = time.perf_counter()
    r = capi.run_case(cfg, collect_history=True)
    dt = time.perf_counter() - t
    print(grid, "converged", r.converged, "steps", r.steps_marched, f"wall {dt:.3f} s",
          f"({dt / max(1, r.steps_marched) * 1e6:.1f} us/iteration)", flush=True)
    cfg = capi.default_config(grid=grid, steps=2000, check_every=1000000)
    t = time.perf_counter()
    r = capi.run_case(cfg)
    dt = time.perf_counter() - t
    print(grid, "fixed 2000 steps, no history:", f"{dt / 2000 * 1e6:.1f} us/iteration", flush=True)
