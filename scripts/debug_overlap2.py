"""np=4 1d-i v3 overlap on one GPU via the block API from 4 host threads;
on failure dump every rank's flags, slot stamps and progress stamps."""
import ctypes as C
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2006_02602_b200 import capi  # noqa: E402

STAGES = ["pack_start", "pack_flag", "wait_start", "wait_done", "unpack_done", "sync_push", "sync_done"]


def dump(b, np_):
    cap = 130 + 16 * np_ + len(STAGES)
    out = (C.c_uint64 * cap)()
    capi.check(b.L.cav_block_debug(b.h, out, cap))
    v = list(out)
    print(f"  rank {b.desc.rank}: flags {v[:4]} stamps {[v[64 + 8 * q + 5] for q in range(2 * np_)]} "
          f"err {[hex(x) for x in v[64 + 16 * np_:66 + 16 * np_]]} "
          f"progress {dict(zip(STAGES, v[130 + 16 * np_:]))}", flush=True)


def trial(strategy, overlap, steps=10, np_=4):
    grid, dims = (20, 16, 16), (4, 1, 1)
    blocks = [capi.Block(r, np_, grid, dims, strategy=strategy, overlap=overlap, timeout_ms=3000)
              for r in range(np_)]
    for b in blocks:
        for r, o in enumerate(blocks):
            if o is not b:
                b.connect(r, ptr=o.arena())
    for b in blocks:
        b.initialize()
    errs = {}
    start = threading.Barrier(np_)

    def go(b):
        start.wait()
        try:
            b.run(steps)
        except Exception as e:
            errs[b.desc.rank] = repr(e)[:100]

    ts = [threading.Thread(target=go, args=(b,)) for b in blocks]
    t = time.time()
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    print(f"{strategy} overlap={overlap} {time.time() - t:.3f}s errors={errs}", flush=True)
    if errs:
        for b in blocks:
            dump(b, np_)
    for b in blocks:
        b.close()
    return not errs


if __name__ == "__main__":
    torch.cuda.init()
    fails = 0
    for rep in range(12):
        for strat in ("v3", "baseline"):
            fails += not trial(strat, True)
    print("failures", fails)
