"""Wider seeded fuzz than tests/test_gpu_fuzz.py (same draw rule), every draw
under the three exchange / ghost variants, against the oracle; prints the
first mismatching draws.  usage: fuzz_wide.py FIRST LAST"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")), "tests"))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402
from oracle.refbind import Oracle  # noqa: E402
from paper_2006_02602_b200 import capi  # noqa: E402
from test_gpu_fuzz import draw  # noqa: E402

first, last = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(first, last):
    kw = draw(seed)
    serial = {k: v for k, v in kw.items() if k not in ("np", "mode", "strategy", "overlap")}
    o = Oracle.run_case(capi.default_config(**serial), collect_fields=True, collect_history=True)
    for env in ({"CAV_STORED_GHOSTS": "-1", "CAV_FUSED_HALO": "1"}, {"CAV_STORED_GHOSTS": "1", "CAV_FUSED_HALO": "1"},
                {"CAV_STORED_GHOSTS": "-1", "CAV_FUSED_HALO": "0"}):
        os.environ.update(env)
        r = capi.run_case(capi.default_config(**kw), collect_fields=True, collect_history=True)
        ok = (list(r.history_iter) == list(o["history_iter"]) and
              np.array_equal(r.history.view(np.uint64), o["history"].view(np.uint64)) and
              np.array_equal(r.fields.view(np.uint64), o["fields"].view(np.uint64)))
        if not ok:
            bad += 1
            print("MISMATCH", seed, env, kw, flush=True)
print(f"fuzz_wide {first}..{last}: {bad} mismatches", flush=True)
