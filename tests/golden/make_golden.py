"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref/libcavity_ref.so,
built by `make -C oracle ref` from /root/reference/proj/src). Run in the build
container: `python tests/golden/make_golden.py`. The fixtures pin both the
plain-C oracle (tests/test_oracle.py) and the GPU path (tests/test_gpu_*.py).

Inputs are drawn with numpy's default_rng (the reference's own tests use
std::mt19937_64, tests/test_kernels.cpp:26-27, which numpy cannot reproduce),
with the reference's value ranges: u,v,w in U(-0.08,0.08), p in U(-2,2),
T in U(299.5,300.5).
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.refbind import Ref, CheckerError, default_config  # noqa: E402
from paper_2006_02602_b200 import _abi as A  # noqa: E402


def hexd(x):
    return float(x).hex()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def random_fields(shape, seed):
    rng = np.random.default_rng(seed)
    f = np.empty((5,) + shape)
    f[0] = rng.uniform(-2.0, 2.0, shape)
    f[1] = rng.uniform(-0.08, 0.08, shape)
    f[2] = rng.uniform(-0.08, 0.08, shape)
    f[3] = rng.uniform(-0.08, 0.08, shape)
    f[4] = rng.uniform(299.5, 300.5, shape)
    return f


def ptrs(f):
    return A.FieldPtrs(*[f[v].ctypes.data for v in range(5)])


def ref_residual(f, n, box, h):
    L = Ref.lib()
    fluid = default_config().fluid
    sp = A.StencilParams()
    L.ref_make_stencil_params(C.c_double(h[0]), C.c_double(h[1]), C.c_double(h[2]), C.byref(fluid),
                              C.byref(sp))
    out = np.zeros_like(f)
    X, Y = n[0] + 4, n[1] + 4
    st = L.ref_residual_box(C.byref(ptrs(f)), C.byref(ptrs(out)), X, Y, C.byref(A.Box.of(*box)),
                            C.byref(sp), 0)
    assert st == 0
    return out


def main():
    out = {}
    # 1. residual kernel on random fields (tests/test_kernels.cpp:77-128 shapes)
    res = {}
    for nx in (5, 9, 12):
        n = (nx, 7, 6)
        f = random_fields((n[2] + 4, n[1] + 4, n[0] + 4), 1000 + nx)
        h = (0.05 / (n[0] - 1), 0.06 / (n[1] - 1), 0.045 / (n[2] - 1))
        box = ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2))
        r = ref_residual(f, n, box, h)
        res[f"in_{nx}"] = f
        res[f"out_{nx}"] = r
        res[f"h_{nx}"] = np.array(h)
    np.savez_compressed(os.path.join(HERE, "residual_random.npz"), **res)

    # 2. full runs: fields + norm histories, bitwise
    cases = {
        "c0_32_1000": dict(grid=(32, 32, 32), steps=1000),
        "r16x12x9_200": dict(grid=(16, 12, 9), steps=200),
        "r10_50_norescale": dict(grid=(10, 10, 10), steps=50, rescale=0),
        "r12_60_cfl07_every7": dict(grid=(12, 12, 12), steps=60, cfl=0.7, check_every=7),
        "conv16_max300": dict(grid=(16, 16, 16), steps=-1, max_steps=300),
        "quiescent_conv": dict(grid=(16, 16, 16), steps=-1, t_hot=300.0, t_cold=300.0),
        "ra1e4_20x16x12_120": dict(grid=(20, 16, 12), steps=120, sigma=None),
    }
    runs = {}
    arrays = {}
    for name, kw in cases.items():
        kw = dict(kw)
        if "sigma" in kw:
            kw.pop("sigma")
            cfg = default_config(**kw)
            cfg.fluid.sigma = cfg.fluid.sigma * 0.1  # Ra = 1e4
        else:
            cfg = default_config(**kw)
        r = Ref.run_case(cfg, collect_fields=True, collect_history=True)
        f = r["fields"]
        runs[name] = {
            "config": kw, "sigma": hexd(cfg.fluid.sigma),
            "steps_marched": int(r["steps_marched"]), "converged": bool(r["converged"]),
            "history_iter": [int(x) for x in r["history_iter"]],
            "history": [[hexd(x) for x in row] for row in r["history"]],
            "fields_sha256": [sha(f[v]) for v in range(5)],
        }
        if f.size <= 5 * 20 * 16 * 12:
            arrays[name] = f
    np.savez_compressed(os.path.join(HERE, "runs_small_fields.npz"), **arrays)

    # 3. error paths (src/runner.cpp:231-233, tests/test_runner.cpp:136-143)
    errors = {}
    for name, kw, hist in [("diverge_cfl50", dict(grid=(16, 16, 16), steps=200, cfl=50.0), False),
                           ("diverge_cfl50_every1", dict(grid=(16, 16, 16), steps=200, cfl=50.0,
                                                         check_every=1), True),
                           ("diverge_12cube", dict(grid=(12, 12, 12), steps=400), False),
                           ("bad_cfl", dict(grid=(8, 8, 8), steps=3, cfl=0.0), False),
                           ("diverge_cfl50_np2", dict(grid=(16, 16, 16), steps=200, cfl=50.0, np=2,
                                                      mode=2), False),
                           ("diverge_cfl50_every1_np2", dict(grid=(16, 16, 16), steps=200, cfl=50.0,
                                                             check_every=1, np=2, mode=2), True),
                           ("diverge_12cube_np2", dict(grid=(12, 12, 12), steps=400, np=2, mode=2),
                            False),
                           ("bad_cfl_np2", dict(grid=(8, 8, 10), steps=3, cfl=0.0, np=2, mode=2),
                            False)]:
        try:
            Ref.run_case(default_config(**kw), collect_history=hist)
            errors[name] = {"config": kw, "history": hist, "error": None}
        except CheckerError as e:
            errors[name] = {"config": kw, "history": hist, "status": e.status, "error": str(e)}

    # 4. host logic tables
    L = Ref.lib()
    tables = {"choose_dims": {}, "partition": {}, "center": {}, "grow": {}, "plans": {},
              "overlap": {}}
    for np_ in (1, 2, 3, 4, 6, 8, 12, 16, 24, 30, 64, 512):
        for mode in range(5):
            d = (C.c_int * 3)()
            st = L.ref_choose_dims(np_, mode, d)
            tables["choose_dims"][f"{np_},{mode}"] = list(d) if st == 0 else None
    for n, dims in [((256, 256, 256), (8, 1, 1)), ((512, 512, 512), (2, 2, 2)),
                    ((512, 512, 512), (1, 2, 4)), ((20, 16, 16), (4, 1, 1)),
                    ((13, 17, 11), (2, 3, 2)), ((32, 32, 32), (2, 2, 2)), ((10, 10, 10), (3, 1, 1))]:
        p = dims[0] * dims[1] * dims[2]
        ext = (C.c_int * (6 * p))()
        st = L.ref_partition(n[0], n[1], n[2], (C.c_int * 3)(*dims), ext)
        key = f"{n}|{dims}"
        tables["partition"][key] = list(ext) if st == 0 else None
        node = (C.c_int * 3)()
        owner = C.c_int()
        if st == 0:
            L.ref_center_owner(n[0], n[1], n[2], (C.c_int * 3)(*dims), node, C.byref(owner))
            tables["center"][key] = list(node) + [owner.value]
    for base in ((256, 256, 256), (32, 32, 32)):
        for np_ in (1, 2, 4, 8, 16, 3):
            for mode in range(5):
                for typ in (1, 2, 3):
                    o = (C.c_int * 3)()
                    st = L.ref_grow_grid(base[0], base[1], base[2], np_, mode, typ, o)
                    tables["grow"][f"{base}|{np_}|{mode}|{typ}"] = list(o) if st == 0 else None
    rng = np.random.default_rng(7)
    for q in range(40):
        n = tuple(int(x) for x in rng.integers(5, 40, 3))
        mask = int(rng.integers(0, 64))
        rank_at = [100 + f if mask & (1 << f) else -1 for f in range(6)]
        for s in range(4):
            ent = (A.PlanEntry * 30)()
            cnt = C.c_int()
            st = L.ref_build_plan(n[0], n[1], n[2], (C.c_int * 6)(*rank_at), s, ent, 30, C.byref(cnt))
            tables["plans"][f"{n}|{mask}|{s}"] = [
                [e.face, e.neighbor, e.nvars, list(e.var)[:e.nvars], list(e.depth)[:e.nvars],
                 e.scalars, e.send_tag, e.recv_tag] for e in ent[:cnt.value]]
    for mask in range(64):
        for n in ((8, 9, 10), (5, 5, 5), (33, 6, 17)):
            rank_at = [100 + f if mask & (1 << f) else -1 for f in range(6)]
            internal = A.Box()
            ext = (A.Box * 6)()
            cnt = C.c_int()
            L.ref_overlap_regions(n[0], n[1], n[2], (C.c_int * 6)(*rank_at), C.byref(internal), ext,
                                  C.byref(cnt))
            tables["overlap"][f"{n}|{mask}"] = [internal.as_tuple()] + [ext[x].as_tuple()
                                                                          for x in range(cnt.value)]
    out = {"runs": runs, "errors": errors, "tables": tables,
           "generator": "tests/golden/make_golden.py via oracle/_ref/libcavity_ref.so "
                        "(reference backend " + L.ref_backend().decode() + ")"}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
