"""Repeat np=4 1d-i overlap runs on one GPU under both comm-stream priorities."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
print("CUDA_DEVICE_MAX_CONNECTIONS", os.environ["CUDA_DEVICE_MAX_CONNECTIONS"], flush=True)

sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2006_02602_b200 import capi  # noqa: E402

torch.cuda.init()
for prio in ("0",):
    os.environ["CAV_COMM_PRIORITY"] = prio
    fails = 0
    for strat in ("baseline", "v3"):
        for rep in range(8):
            cfg = capi.default_config(grid=(20, 16, 16), steps=10, np=4, mode="1d-i", strategy=strat,
                                      overlap=1, timeout_ms=3000)
            t = time.time()
            try:
                capi.run_case(cfg, collect_fields=True)
            except Exception as e:
                fails += 1
                print(f"prio={prio} {strat} rep={rep} {time.time()-t:.3f}s {repr(e)[:110]}", flush=True)
    print(f"prio={prio}: {fails} failures of 24", flush=True)
