# diagnostics: field statistics after N iterations at 256^3 (env selects variant)
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
import torch
from paper_2006_02602_b200 import capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1))
b.initialize()
b.run(n)
f = b.download()
for v, nm in enumerate("puvwT"):
    x = f[v][2:-2, 2:-2, 2:-2]
    fin = np.isfinite(x)
    ax = np.abs(x[fin]) if fin.any() else np.zeros(1)
    nz = np.count_nonzero(x[fin] - (300.0 if nm == "T" else 0.0))
    print(os.environ.get("CAV_EXP", "0"), nm, "nonfinite", int((~fin).sum()), "max|x|", float(ax.max()),
          "nonzero(pert)", nz, "tiny(<1e-300)", int(((ax > 0) & (ax < 1e-300)).sum()))
b.close()
