"""ctypes mirror of include/cavity_b200.h (structs and enums only, no loading).

Kept in one place so the product wrapper (`capi.py`) and the test-side
checkers under tests agree on the exact C layout.
"""
import ctypes as C

CAV_OK, CAV_EINVAL, CAV_ERUNTIME, CAV_ELOGIC, CAV_ELENGTH, CAV_ECUDA, CAV_ETIMEOUT = range(7)

MODES = {"1d-i": 0, "1d-j": 1, "1d-k": 2, "2d": 3, "3d": 4}
MODE_NAMES = {v: k for k, v in MODES.items()}
STRATEGIES = {"baseline": 0, "v1": 1, "v2": 2, "v3": 3}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
VAR_NAMES = ("p", "u", "v", "w", "T")
WALL = -1


class Box(C.Structure):
    _fields_ = [("lo", C.c_int * 3), ("hi", C.c_int * 3)]

    @classmethod
    def of(cls, lo, hi):
        b = cls()
        for a in range(3):
            b.lo[a] = lo[a]
            b.hi[a] = hi[a]
        return b

    def as_tuple(self):
        return (tuple(self.lo), tuple(self.hi))


class StencilParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "inv2dx", "inv2dy", "inv2dz", "invdx2", "invdy2", "invdz2", "invdx4", "invdy4",
        "invdz4", "kdx3", "kdy3", "kdz3", "u_ref", "nu", "alpha", "rho", "inv_rho", "sigma",
        "t_inf", "gx", "gy", "gz")]


class FluidParams(C.Structure):
    _fields_ = [("rho", C.c_double), ("nu", C.c_double), ("alpha", C.c_double),
                ("sigma", C.c_double), ("gravity", C.c_double * 3), ("u_ref", C.c_double),
                ("kappa", C.c_double), ("t_hot", C.c_double), ("t_cold", C.c_double),
                ("t_inf", C.c_double), ("length", C.c_double)]


class FieldPtrs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("p", "u", "v", "w", "t")]


NORM_WORDS = 360  # CAV_NORM_WORDS: 5 x 70 digits, 5 L-inf bit patterns, padding


class PlanEntry(C.Structure):
    _fields_ = [("face", C.c_int), ("neighbor", C.c_int), ("nvars", C.c_int),
                ("var", C.c_int * 5), ("depth", C.c_int * 5), ("scalars", C.c_longlong),
                ("send_tag", C.c_int), ("recv_tag", C.c_int)]


class RunConfig(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("np", C.c_int),
                ("mode", C.c_int), ("dims", C.c_int * 3), ("strategy", C.c_int),
                ("overlap", C.c_int), ("steps", C.c_longlong), ("fluid", FluidParams),
                ("cfl", C.c_double), ("max_steps", C.c_longlong), ("conv_tol", C.c_double),
                ("rescale", C.c_int), ("check_every", C.c_int), ("seed", C.c_uint64),
                ("timeout_ms", C.c_double), ("monitor_every", C.c_int),
                ("verify_tol", C.c_double), ("devices", C.c_int * 8)]


class CaseOptions(C.Structure):
    _fields_ = [("collect_fields", C.c_int), ("collect_history", C.c_int),
                ("corrupt_exchange", C.c_int)]


class Ledger(C.Structure):
    _fields_ = [("face_bytes", C.c_uint64 * 6), ("face_messages", C.c_uint64 * 6),
                ("last_face_bytes", C.c_uint64 * 6), ("bytes_sent", C.c_uint64),
                ("messages_sent", C.c_uint64), ("exchanges", C.c_uint64)]

    def as_dict(self):
        return {"face_bytes": list(self.face_bytes), "face_messages": list(self.face_messages),
                "last_face_bytes": list(self.last_face_bytes), "bytes_sent": self.bytes_sent,
                "messages_sent": self.messages_sent, "exchanges": self.exchanges}


class CaseResultC(C.Structure):
    _fields_ = [("steps_marched", C.c_longlong), ("steps_timed", C.c_longlong),
                ("converged", C.c_int), ("np", C.c_int), ("dims", C.c_int * 3),
                ("wall_time_s", C.c_double), ("ssspnt", C.c_double), ("bytes_sent", C.c_uint64),
                ("fields", C.POINTER(C.c_double)), ("hist_capacity", C.c_longlong),
                ("hist_count", C.c_longlong), ("hist_iter", C.POINTER(C.c_longlong)),
                ("hist_l2", C.POINTER(C.c_double)), ("ledger_capacity", C.c_int),
                ("ledgers", C.POINTER(Ledger)), ("hist_linf", C.POINTER(C.c_double))]


class BlockDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("np", C.c_int), ("gnx", C.c_int), ("gny", C.c_int),
                ("gnz", C.c_int), ("dims", C.c_int * 3), ("strategy", C.c_int),
                ("overlap", C.c_int), ("fluid", FluidParams), ("cfl", C.c_double),
                ("rescale", C.c_int), ("corrupt_exchange", C.c_int), ("device", C.c_int),
                ("timeout_ms", C.c_double), ("jitter_seed", C.c_uint64)]


class RunIO(C.Structure):
    _fields_ = [("first_it", C.c_longlong), ("n_its", C.c_longlong), ("check_every", C.c_int),
                ("want_norms", C.c_int), ("norm_digits", C.POINTER(C.c_uint64)),
                ("check_iters", C.POINTER(C.c_longlong)), ("n_checks", C.c_longlong),
                ("err_iteration", C.c_longlong), ("err_kind", C.c_int),
                ("seconds", C.c_double), ("ledger", Ledger),
                ("device_conv", C.c_int), ("conv_tol", C.c_double), ("conv_peaks", C.c_double * 5),
                ("conv_iter", C.c_longlong)]


def apply_overrides(cfg, **kw):
    """Set RunConfig fields by name; fluid constants may be given flat
    (nu=..., t_hot=...), grid as a 3-tuple, mode/strategy as names."""
    for k, v in kw.items():
        if k == "grid":
            cfg.nx, cfg.ny, cfg.nz = v
        elif k == "mode":
            cfg.mode = MODES[v] if isinstance(v, str) else v
        elif k == "strategy":
            cfg.strategy = STRATEGIES[v] if isinstance(v, str) else v
        elif k == "dims":
            for a in range(3):
                cfg.dims[a] = v[a]
        elif k == "devices":
            for a in range(8):
                cfg.devices[a] = v[a % len(v)]
        elif k == "gravity":
            for a in range(3):
                cfg.fluid.gravity[a] = v[a]
        elif k in ("rho", "nu", "alpha", "sigma", "u_ref", "kappa", "t_hot", "t_cold", "t_inf",
                   "length"):
            setattr(cfg.fluid, k, v)
        else:
            if not hasattr(cfg, k):
                raise AttributeError("RunConfig has no field " + k)
            setattr(cfg, k, v)
    return cfg
