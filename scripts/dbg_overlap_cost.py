# Relative cost of the overlap path (internal TMA box + pointwise shells) vs
# exchange-then-full-box, for in-process ranks sharing one GPU (their kernels
# serialise, so the difference is the extra work, not the hidden exchange).
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
for np_, mode in ((1, "3d"), (2, "3d"), (8, "3d"), (4, "1d-i")):
    for ov in ((0, 1) if np_ > 1 else (0,)):
        cfg = capi.default_config(grid=(256, 256, 256), steps=60, np=np_, mode=mode, strategy="v3", overlap=ov)
        r = capi.run_case(cfg)
        print(f"np={np_} {mode} overlap={ov}: {r.wall_time_s / r.steps_timed * 1e3:.3f} ms/iteration "
              f"(all ranks on one GPU)", flush=True)
