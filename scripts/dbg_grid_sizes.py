# Per-iteration time of fixed-step runs (no norms) over grid sizes, for the
# current environment's step configuration (e.g. CAV_STORED_GHOSTS=0/1), and
# one solve to convergence at 32^3.
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
tag = os.environ.get("TAG", "")
for n in (32, 64, 128, 256):
    b = capi.Block(0, 1, (n, n, n), (1, 1, 1))
    b.initialize()
    b.run(20)
    its = 2000 if n <= 64 else 500
    t0 = time.perf_counter()
    b.run(its)
    t = time.perf_counter() - t0
    print(f"{tag} n={n}: {t / its * 1e6:.1f} us/iteration", flush=True)
    b.close()
cfg = capi.default_config(grid=(32, 32, 32), steps=-1)
t0 = time.perf_counter()
r = capi.run_case(cfg)
print(f"{tag} solve 32^3: {r.steps_marched} iterations, {time.perf_counter() - t0:.3f} s", flush=True)
