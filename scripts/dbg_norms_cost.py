# Cost of the residual-norm (check) iterations: 256^3, 500 iterations with
# norms every 10 (cavity solve cadence) vs none (run_bench cadence).
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1))
b.initialize()
b.run(20)
for want, every in ((False, 10), (True, 10), (True, 1)):
    t0 = time.perf_counter()
    secs, chk = b.run(500, check_every=every, want_norms=want)
    t = time.perf_counter() - t0
    print(f"norms={want} every={every}: {t / 500 * 1e3:.3f} ms/iteration ({len(chk)} checks)", flush=True)
b.close()
