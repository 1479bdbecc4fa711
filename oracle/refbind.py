"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU checkers.

* `Ref`    — the unmodified reference (oracle/_ref/libcavity_ref.so, built by
             oracle/Makefile from /root/reference/proj/src + ref_driver.cpp).
* `Oracle` — the plain-C restatement (oracle/_build/libcavity_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module; the product path never does.
"""
import ctypes as C
import os

import numpy as np

from paper_2006_02602_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcavity_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libcavity_oracle.so")

_P = C.c_void_p


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


class CheckerError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def ref_available():
    return os.path.exists(REF_SO)


def default_config(**kw):
    """RunConfig defaults (include/cavity/util/config.hpp:15-34) with overrides."""
    lib = Ref.lib() if ref_available() else Oracle.lib()
    cfg = A.RunConfig()
    (lib.ref_run_config_default if lib is Ref._lib else lib.oc_run_config_default)(C.byref(cfg))
    return apply_overrides(cfg, **kw)


apply_overrides = A.apply_overrides


def _run(fn, errfn, cfg, collect_fields, collect_history, corrupt=False):
    n = cfg.nx * cfg.ny * cfg.nz
    fields = np.zeros(5 * n) if collect_fields else None
    target = cfg.steps if cfg.steps >= 0 else cfg.max_steps
    cap = int(target // max(1, cfg.check_every) + 2)
    hist_iter = np.zeros(cap, dtype=np.int64)
    hist_l2 = np.zeros(5 * cap)
    led = (A.Ledger * max(1, cfg.np))()
    out = A.CaseResultC()
    out.fields = fields.ctypes.data_as(C.POINTER(C.c_double)) if fields is not None else None
    out.hist_capacity = cap
    out.hist_iter = hist_iter.ctypes.data_as(C.POINTER(C.c_longlong))
    out.hist_l2 = hist_l2.ctypes.data_as(C.POINTER(C.c_double))
    out.ledger_capacity = max(1, cfg.np)
    out.ledgers = C.cast(led, C.POINTER(A.Ledger))
    opt = A.CaseOptions(int(collect_fields), int(collect_history), int(corrupt))
    st = fn(C.byref(cfg), C.byref(opt), C.byref(out))
    if st != 0:
        raise CheckerError(st, errfn().decode())
    h = int(out.hist_count)
    res = {
        "steps_marched": out.steps_marched, "steps_timed": out.steps_timed,
        "converged": bool(out.converged), "np": out.np, "dims": tuple(out.dims),
        "wall_time_s": out.wall_time_s, "ssspnt": out.ssspnt, "bytes_sent": out.bytes_sent,
        "history_iter": hist_iter[:h].copy(), "history": hist_l2[:5 * h].reshape(h, 5).copy(),
        "ledgers": [led[r].as_dict() for r in range(out.np if out.np > 0 else 0)],
    }
    if fields is not None:
        res["fields"] = fields.reshape(5, cfg.nz, cfg.ny, cfg.nx)
    return res


class Ref:
    """The real reference, through oracle/_ref/libcavity_ref.so."""
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ref_available():
                raise FileNotFoundError(REF_SO + " not built (make -C oracle ref)")
            lib = C.CDLL(REF_SO)
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_backend.restype = C.c_char_p
            lib.ref_repro_sum.restype = C.c_double
            lib.ref_repro_value.restype = C.c_double
            cls._lib = lib
        return cls._lib

    @classmethod
    def run_case(cls, cfg, collect_fields=True, collect_history=False, corrupt=False):
        lib = cls.lib()
        return _run(lib.ref_run_case, lib.ref_last_error, cfg, collect_fields, collect_history,
                    corrupt)


class Oracle:
    """The plain-C restatement, through oracle/_build/libcavity_oracle.so."""
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise FileNotFoundError(ORACLE_SO + " not built (make -C oracle oracle)")
            lib = C.CDLL(ORACLE_SO)
            lib.oc_last_error.restype = C.c_char_p
            lib.oc_repro_value.restype = C.c_double
            cls._lib = lib
        return cls._lib

    @classmethod
    def run_case(cls, cfg, collect_fields=True, collect_history=False):
        """Serial (np=1) restatement of run_case; the reference is bitwise
        decomposition-independent (P/README.md:10-15), so this is the field
        and history oracle for every np/strategy/overlap."""
        lib = cls.lib()
        return _run(lib.oc_run_serial, lib.oc_last_error, cfg, collect_fields, collect_history)
