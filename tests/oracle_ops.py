"""Test helpers: the plain-C oracle's op-level functions on numpy storage
(Field3 layout, arrays shaped (5, nz+4, ny+4, nx+4)). Checker only."""
import ctypes as C

import numpy as np

from oracle.refbind import Oracle
from paper_2006_02602_b200 import _abi as A


def _fp(f):
    return A.FieldPtrs(*[f[v].ctypes.data for v in range(5)])


def random_fields(n, seed, vel=0.08):
    rng = np.random.default_rng(seed)
    shape = (n[2] + 4, n[1] + 4, n[0] + 4)
    f = np.empty((5,) + shape)
    f[0] = rng.uniform(-2.0, 2.0, shape)
    for v in (1, 2, 3):
        f[v] = rng.uniform(-vel, vel, shape)
    f[4] = rng.uniform(299.5, 300.5, shape)
    return f


def stencil(h, fluid):
    sp = A.StencilParams()
    Oracle.lib().oc_make_stencil_params(C.c_double(h[0]), C.c_double(h[1]), C.c_double(h[2]),
                                        C.byref(fluid), C.byref(sp))
    return sp


def residual(f, n, box, sp):
    out = np.zeros_like(f)
    Oracle.lib().oc_residual_box(C.byref(_fp(f)), C.byref(_fp(out)), n[0] + 4, n[1] + 4,
                                 C.byref(A.Box.of(*box)), C.byref(sp))
    return out


def update(q, r, dt, n, box):
    q = q.copy()
    Oracle.lib().oc_update_box(q.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                               C.c_double(dt), n[0] + 4, n[1] + 4, C.byref(A.Box.of(*box)))
    return q


def bc(f, n, walls, fluid):
    f = f.copy()
    w = (C.c_int * 6)(*[int(x) for x in walls])
    Oracle.lib().oc_apply_bc(C.byref(_fp(f)), n[0], n[1], n[2], w, C.byref(fluid))
    return f


def compute_dt(f, n, h, fluid, cfl):
    dt = C.c_double()
    st = Oracle.lib().oc_compute_dt(C.byref(_fp(f)), n[0], n[1], n[2], C.c_double(h[0]),
                                    C.c_double(h[1]), C.c_double(h[2]), C.byref(fluid),
                                    C.c_double(cfl), C.byref(dt))
    if st:
        raise RuntimeError(Oracle.lib().oc_last_error().decode())
    return dt.value


def rescale(p, n, pc):
    p = p.copy()
    Oracle.lib().oc_rescale(p.ctypes.data_as(C.c_void_p), n[0], n[1], n[2], C.c_double(pc))
    return p


def norm_limbs(r, n):
    out = np.zeros(350, dtype=np.uint64)
    st = Oracle.lib().oc_norm_partials(C.byref(_fp(r)), n[0], n[1], n[2],
                                       out.ctypes.data_as(C.POINTER(C.c_uint64)))
    if st:
        raise ValueError(Oracle.lib().oc_last_error().decode())
    return out.reshape(5, 70)


def copy_box_to(f1, n, box):
    b = A.Box.of(*box)
    vol = int(np.prod([box[1][a] - box[0][a] for a in range(3)]))
    out = np.zeros(vol)
    Oracle.lib().oc_copy_box_to(f1.ctypes.data_as(C.c_void_p), n[0] + 4, n[1] + 4, C.byref(b),
                                out.ctypes.data_as(C.c_void_p))
    return out


def march(f, n, h, fluid, cfl, steps, walls=(1, 1, 1, 1, 1, 1), center=None, rescale_on=True):
    """rank_main's loop for one block from an arbitrary state (serial, no
    exchange): BC, residual, dt, update, centre rescale."""
    f = np.ascontiguousarray(f).copy()
    sp = stencil(h, fluid)
    box = ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2))
    if center is None:
        center = tuple((x - 1) // 2 + 2 for x in n)
    for _ in range(steps):
        f = bc(f, n, walls, fluid)
        r = residual(f, n, box, sp)
        dt = compute_dt(f, n, h, fluid, cfl)
        for v in range(5):
            f[v] = update(f[v], r[v], dt, n, box)
        if rescale_on:
            pc = f[0][center[2], center[1], center[0]]
            f[0] = rescale(f[0], n, pc)
    return f
