"""Repeat the np=4 1d-i v2 overlap case on one GPU, timing each run."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2006_02602_b200 import capi  # noqa: E402

torch.cuda.init()
for kern in ("tma", "tiled"):
    os.environ["CAV_STEP_KERNEL"] = kern
    for strat in ("baseline", "v1", "v2", "v3"):
        for ov in (0, 1):
            for rep in range(3):
                cfg = capi.default_config(grid=(20, 16, 16), steps=10, np=4, mode="1d-i", strategy=strat,
                                          overlap=ov, timeout_ms=4000)
                t = time.time()
                try:
                    capi.run_case(cfg, collect_fields=True)
                    res = "ok"
                except Exception as e:
                    res = repr(e)[:120]
                print(f"{kern} {strat} ov={ov} rep={rep} {time.time()-t:.3f}s {res}", flush=True)
