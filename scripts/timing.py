"""Timing probes of the hot path on one GPU (results to stdout):

  python scripts/timing.py grids      per-iteration time over grid sizes (fixed steps)
  python scripts/timing.py norms      cost of norm (check) iterations at 256^3
  python scripts/timing.py ranks      in-process ranks sharing one GPU (the multi-rank
                                      path's extra work: their kernels serialise, so
                                      the sum over ranks is compared with one rank)
  python scripts/timing.py solve      32^3 to convergence
  python scripts/timing.py runs       per-iteration time of run_case (fixed steps, one rank) by grid size

Every number is device time from cav_block_bench / run_case's own timer.
"""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from paper_2006_02602_b200 import capi  # noqa: E402


def grids():
    for n in (32, 64, 128, 256, 512):
        b = capi.Block(0, 1, (n, n, n), (1, 1, 1))
        b.initialize()
        b.run(20)
        its = 2000 if n <= 64 else (500 if n <= 256 else 100)
        total, step, _ = b.bench(its)
        print(f"n={n}: {total / its * 1e3:.1f} us/iteration, step kernel {step * 1e3:.1f} us, "
              f"{n ** 3 * its / (total * 1e-3) / 1e6:.0f} MCUPS", flush=True)
        b.close()


def norms():
    b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1))
    b.initialize()
    b.run(20)
    for want, every in ((False, 10), (True, 10), (True, 1)):
        secs, chk = b.run(500, check_every=every, want_norms=want)
        print(f"norms={want} every={every}: {secs / 500 * 1e3:.3f} ms/iteration ({len(chk)} checks)", flush=True)
    b.close()


def ranks():
    its = int(os.environ.get("ITS", "60"))
    for grid, np_, mode in (((256,) * 3, 1, "3d"), ((256,) * 3, 2, "3d"), ((256,) * 3, 8, "3d"),
                            ((256,) * 3, 4, "1d-i"), ((512,) * 3, 1, "3d"), ((512,) * 3, 8, "3d"),
                            ((512,) * 3, 8, "2d")):
        for ov in ((0, 1) if np_ > 1 else (0,)):
            cfg = capi.default_config(grid=grid, steps=its, np=np_, mode=mode, strategy="v3", overlap=ov)
            r = capi.run_case(cfg)
            print(f"{grid[0]}^3 np={np_} {mode} overlap={ov}: {r.wall_time_s / r.steps_timed * 1e3:.3f} ms/iteration "
                  f"(all ranks on one GPU)", flush=True)


def runs():
    for n in (32, 64, 128, 256):
        its = 4000 if n <= 64 else (1000 if n <= 128 else 400)
        r = capi.run_case(capi.default_config(grid=(n, n, n), steps=its))
        print(f"n={n}: {r.wall_time_s / r.steps_timed * 1e6:.1f} us/iteration (run_case, {its} steps)", flush=True)


def solve():
    cfg = capi.default_config(grid=(32, 32, 32), steps=-1)
    t0 = time.perf_counter()
    r = capi.run_case(cfg)
    print(f"solve 32^3: {r.steps_marched} iterations, {time.perf_counter() - t0:.3f} s", flush=True)


if __name__ == "__main__":
    for what in sys.argv[1:] or ["grids", "norms", "ranks", "solve"]:
        globals()[what]()
