"""Two in-process ranks on one GPU, driven from two host threads; dumps the
exchange arenas after the run (flags, scalar-slot stamps, error codes)."""
import ctypes as C
import sys
import threading

import numpy as np

sys.path.insert(0, ".")
from paper_2006_02602_b200 import capi  # noqa: E402


def dump(b, np_):
    cap = 64 + 16 * np_ + 2 + 64
    out = (C.c_uint64 * cap)()
    capi.check(b.L.cav_block_debug(b.h, out, cap))
    v = list(out)
    flags = v[:8]
    slots = [v[64 + 8 * q: 64 + 8 * q + 8] for q in range(2 * np_)]
    err = v[64 + 16 * np_: 66 + 16 * np_]
    cnt = v[66 + 16 * np_: 66 + 16 * np_ + 8]
    print("  flags", flags)
    print("  slot stamps", [s[5] for s in slots])
    print("  err", [hex(x) for x in err], "counters", cnt, flush=True)


def trial(grid, dims, overlap, steps=3):
    np_ = dims[0] * dims[1] * dims[2]
    print(f"== grid {grid} dims {dims} overlap {overlap}", flush=True)
    blocks = [capi.Block(r, np_, grid, dims, strategy="v3", overlap=overlap, timeout_ms=3000)
              for r in range(np_)]
    for b in blocks:
        for r, o in enumerate(blocks):
            if o is not b:
                b.connect(r, ptr=o.arena())
    for b in blocks:
        b.initialize()
    errs = {}

    def go(b):
        try:
            b.run(steps)
        except Exception as e:  # report and keep going
            errs[b.desc.rank] = repr(e)

    ts = [threading.Thread(target=go, args=(b,)) for b in blocks]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    print("  errors:", errs, flush=True)
    for b in blocks:
        print(" rank", b.desc.rank)
        dump(b, np_)
    for b in blocks:
        b.close()


if __name__ == "__main__":
    import torch
    torch.cuda.init()
    trial((16, 16, 16), (1, 1, 2), False)
    trial((16, 16, 16), (1, 1, 2), True)
    trial((20, 16, 16), (2, 1, 1), False)
