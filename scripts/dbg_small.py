import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
cfg = capi.default_config(grid=(24, 20, 16), steps=3, check_every=5)
r = capi.run_case(cfg, collect_fields=True, collect_history=True)
print("ok", r.history[:2])
