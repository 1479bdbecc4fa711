# Per-call overhead of cav_block_run segments (the convergence driver runs one
# segment per check): 32^3, 10 iterations per call, with and without norms.
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (32, 32, 32), (1, 1, 1))
b.initialize()
b.run(10)
for want in (False, True, False, True):
    t = time.perf_counter()
    for _ in range(100):
        b.run(10, check_every=10, want_norms=want)
    dt = (time.perf_counter() - t) / 100
    print(f"norms={want}: {dt * 1e6:.1f} us per 10-iteration segment", flush=True)
t = time.perf_counter()
b.run(1000, check_every=10, want_norms=True)
print(f"one call, 1000 its, norms every 10: {(time.perf_counter() - t) / 100 * 1e6:.1f} us per 10 iterations")
b.close()
