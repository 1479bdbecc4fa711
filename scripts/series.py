"""GPU strong/weak scaling series in the reference's RunRecord CSV
(bench --scaling strong|weak, /root/reference/proj/src/bench.cpp) plus the
B200 sidecar (roofline fraction, exposed communication, GPUs shared).

  python scripts/series.py OUT_DIR [--steps K] [--which c2,c3,c4]

c2: 256^3, 1d-i, np 1/2/4/8 (strong)      BASELINE configs[2]
c3: 512^3, 2d and 3d, np 1/2/4/8 (strong) BASELINE configs[3]
c4: 256^3 per rank, 3d, np 1/2/4/8 (weak, grow_grid type 2) BASELINE configs[4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from paper_2006_02602_b200 import series  # noqa: E402

CASES = {
    "c2": dict(grid=(256, 256, 256), modes=["1d-i"], scaling="strong"),
    "c3": dict(grid=(512, 512, 512), modes=["2d", "3d"], scaling="strong"),
    "c4": dict(grid=(256, 256, 256), modes=["3d"], scaling="weak"),
}

if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("out")
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--which", default="c2,c3,c4")
    p.add_argument("--np", default="1,2,4,8")
    a = p.parse_args()
    nps = [int(x) for x in a.np.split(",")]
    for name in a.which.split(","):
        c = CASES[name]
        ser, extra, warn = series.run_series(c["grid"], nps, c["modes"], scaling=c["scaling"], steps=a.steps,
                                             warmup=a.warmup)
        paths = series.write_outputs(ser, extra, os.path.join(a.out, name), c["scaling"])
        for w in warn:
            print("warning:", w)
        for e in extra:
            print(name, e, flush=True)
        print(name, "->", paths, flush=True)
