"""Python face of the C ABI (include/cavity_b200.h).

Mirrors the reference's driver API (/root/reference/proj/include/cavity/
runner.hpp:36-52): `run_case`, `compare_fields`, `verify_against_serial`,
plus the op-level kernels:: seam and the host-side decomposition helpers.
Every compute call goes to the in-tree sm_100a library
`paper_2006_02602_b200/lib/libcavity_b200.so`; there is no CPU fallback —
if the library is missing, `lib()` raises.
"""
import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi as A

# Several in-process ranks may share one GPU (tests); each drives two streams
# whose kernels wait on each other, so the streams must not share hardware
# queues. Effective only if set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_NAME = "libcavity_b200.so"
LIB_FMAD_NAME = "libcavity_b200_fmad.so"


class CavityError(RuntimeError):
    status = A.CAV_ERUNTIME


class InvalidArgument(CavityError, ValueError):  # std::invalid_argument
    status = A.CAV_EINVAL


class LogicError(CavityError):  # std::logic_error
    status = A.CAV_ELOGIC


class LengthError(CavityError):  # std::length_error
    status = A.CAV_ELENGTH


class CudaError(CavityError):
    status = A.CAV_ECUDA


class TransportTimeout(CavityError):  # transport::TransportTimeout
    status = A.CAV_ETIMEOUT


_ERRORS = {A.CAV_EINVAL: InvalidArgument, A.CAV_ERUNTIME: CavityError, A.CAV_ELOGIC: LogicError,
           A.CAV_ELENGTH: LengthError, A.CAV_ECUDA: CudaError, A.CAV_ETIMEOUT: TransportTimeout}

_libs = {}

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_LL = C.c_longlong


def lib_path(fmad=False):
    # CAV_LIB: an alternate build of the same library (A/B timing of two builds in one run)
    alt = os.environ.get("CAV_LIB")
    if alt and not fmad:
        return alt
    return os.path.join(LIB_DIR, LIB_FMAD_NAME if fmad else LIB_NAME)


def lib(fmad=False):
    """The sm_100a library. Raises if it was not built — no fallback."""
    if fmad not in _libs:
        path = lib_path(fmad)
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with __graft_entry__.build() "
                              "(make -C paper_2006_02602_b200/csrc)")
        L = C.CDLL(path)
        L.cav_last_error.restype = C.c_char_p
        L.cav_version.restype = C.c_char_p
        L.cav_repro_value.restype = C.c_double
        L.cav_repro_value.argtypes = [C.POINTER(C.c_uint64)]
        L.cav_residual_box.argtypes = [C.POINTER(A.FieldPtrs), C.POINTER(A.FieldPtrs), _I, _I,
                                       C.POINTER(A.Box), C.POINTER(A.StencilParams), _P]
        L.cav_update_box.argtypes = [_P, _P, _D, _I, _I, C.POINTER(A.Box), _P]
        L.cav_apply_boundary_conditions.argtypes = [C.POINTER(A.FieldPtrs), _I, _I, _I,
                                                    C.POINTER(_I), C.POINTER(A.FluidParams), _P]
        L.cav_compute_dt.argtypes = [C.POINTER(A.FieldPtrs), _I, _I, _I, _D, _D, _D,
                                     C.POINTER(A.FluidParams), _D, C.POINTER(_D), _P]
        L.cav_rescale_pressure.argtypes = [_P, _I, _I, _I, _D, _P]
        L.cav_residual_norm_partials.argtypes = [C.POINTER(A.FieldPtrs), _I, _I, _I,
                                                 C.POINTER(C.c_uint64), _P]
        L.cav_copy_box_to.argtypes = [_P, _I, _I, C.POINTER(A.Box), _P, _P]
        L.cav_copy_box_from.argtypes = [_P, _I, _I, C.POINTER(A.Box), _P, _P]
        L.cav_block_bench.argtypes = [_P, _LL, C.POINTER(_D)]
        _libs[fmad] = L
    return _libs[fmad]


def check(st, L=None):
    if st != A.CAV_OK:
        L = L or lib()
        raise _ERRORS.get(st, CavityError)(L.cav_last_error().decode())


def version(fmad=False):
    return lib(fmad).cav_version().decode()


# ---- configuration -----------------------------------------------------------

def default_config(**kw):
    """RunConfig defaults (include/cavity/util/config.hpp:15-34) plus overrides."""
    cfg = A.RunConfig()
    lib().cav_run_config_default(C.byref(cfg))
    return A.apply_overrides(cfg, **kw)


def fluid_for_rayleigh(ra):
    f = A.FluidParams()
    lib().cav_fluid_for_rayleigh(C.c_double(ra), C.byref(f))
    return f


def stencil_params(dx, dy, dz, fluid):
    sp = A.StencilParams()
    lib().cav_make_stencil_params(_D(dx), _D(dy), _D(dz), C.byref(fluid), C.byref(sp))
    return sp


def cavity_spacing(n, length=0.05):
    h = (C.c_double * 3)()
    check(lib().cav_make_cavity_grid(n[0], n[1], n[2], _D(length), _D(length), _D(length), h))
    return tuple(h)


# ---- run level (include/cavity/runner.hpp) -----------------------------------

@dataclass
class CaseResult:
    """CaseResult (include/cavity/runner.hpp:20-29) plus the record fields."""
    steps_marched: int
    steps_timed: int
    converged: bool
    np: int
    dims: tuple
    wall_time_s: float
    ssspnt: float
    bytes_sent: int
    history_iter: np.ndarray
    history: np.ndarray
    ledgers: List[dict]
    fields: Optional[np.ndarray] = None  # (5, nz, ny, nx): p,u,v,w,T
    history_linf: Optional[np.ndarray] = None  # (samples, 5): max |R_v| per check iteration

    def __getitem__(self, k):  # dict-style access, like the oracle results
        return getattr(self, k)


def run_case(cfg, collect_fields=False, collect_history=False, corrupt_exchange=False, fmad=False):
    """run_case (src/runner.cpp:259-338) on the GPU(s) in cfg.devices.
    fmad=True uses the tolerance build (FMA contraction; not bitwise)."""
    n = cfg.nx * cfg.ny * cfg.nz
    fields = np.zeros(5 * n) if collect_fields else None
    target = cfg.steps if cfg.steps >= 0 else cfg.max_steps
    cap = int(target // max(1, cfg.check_every) + 2)
    hist_iter = np.zeros(cap, dtype=np.int64)
    hist_l2 = np.zeros(5 * cap)
    hist_linf = np.zeros(5 * cap)
    nl = max(1, cfg.np)
    led = (A.Ledger * nl)()
    out = A.CaseResultC()
    out.fields = fields.ctypes.data_as(C.POINTER(C.c_double)) if fields is not None else None
    out.hist_capacity = cap
    out.hist_iter = hist_iter.ctypes.data_as(C.POINTER(C.c_longlong))
    out.hist_l2 = hist_l2.ctypes.data_as(C.POINTER(C.c_double))
    out.hist_linf = hist_linf.ctypes.data_as(C.POINTER(C.c_double))
    out.ledger_capacity = nl
    out.ledgers = C.cast(led, C.POINTER(A.Ledger))
    opt = A.CaseOptions(int(collect_fields), int(collect_history), int(corrupt_exchange))
    L = lib(fmad)
    check(L.cav_run_case(C.byref(cfg), C.byref(opt), C.byref(out)), L)
    h = int(out.hist_count)
    return CaseResult(
        steps_marched=out.steps_marched, steps_timed=out.steps_timed,
        converged=bool(out.converged), np=out.np, dims=tuple(out.dims),
        wall_time_s=out.wall_time_s, ssspnt=out.ssspnt, bytes_sent=out.bytes_sent,
        history_iter=hist_iter[:h].copy(), history=hist_l2[:5 * h].reshape(h, 5).copy(),
        ledgers=[led[r].as_dict() for r in range(out.np)],
        fields=fields.reshape(5, cfg.nz, cfg.ny, cfg.nx) if fields is not None else None,
        history_linf=hist_linf[:5 * h].reshape(h, 5).copy())


@dataclass
class VerifyReport:
    """VerifyReport (include/cavity/runner.hpp:31-38)."""
    passed: bool = False
    tol: float = 0.0
    steps: int = 0
    max_abs: List[float] = field(default_factory=lambda: [0.0] * 5)
    rel: List[float] = field(default_factory=lambda: [0.0] * 5)

    def summary(self):
        lines = [f"  {n:<2s} max|diff| = {a:.3e}   rel = {r:.3e}"
                 for n, a, r in zip(A.VAR_NAMES, self.max_abs, self.rel)]
        lines.append(f"verify: {'PASS' if self.passed else 'FAIL'} (tolerance {self.tol:.1e}, "
                     f"{self.steps} steps)")
        return "\n".join(lines)


def compare_fields(ref, test, tol):
    """compare_fields (src/runner.cpp:355-375): per variable max|diff| and
    max|diff| / max(|ref|,|test|) over the global interior."""
    ref = np.asarray(ref)
    test = np.asarray(test)
    if ref.shape != test.shape:
        raise InvalidArgument("verify: grid sizes differ")
    rep = VerifyReport(passed=True, tol=tol)
    for v in range(5):
        a, b = ref[v].ravel(), test[v].ravel()
        max_abs = float(np.max(np.abs(a - b))) if a.size else 0.0
        scale = float(max(np.max(np.abs(a)), np.max(np.abs(b)))) if a.size else 0.0
        rep.max_abs[v] = max_abs
        rep.rel[v] = max_abs / scale if scale > 0.0 else max_abs
        if not (rep.rel[v] <= tol):
            rep.passed = False
    return rep


def verify_against_serial(cfg, corrupt_exchange=False):
    """verify_against_serial (src/runner.cpp:377-396): run cfg, then the same
    physics on one rank, compare the fields."""
    if cfg.steps < 0:
        raise InvalidArgument("verify: a fixed step count is required (--steps)")
    test = run_case(cfg, collect_fields=True, corrupt_exchange=corrupt_exchange)
    serial = A.RunConfig.from_buffer_copy(cfg)
    serial.np = 1
    serial.dims[0] = serial.dims[1] = serial.dims[2] = 1
    serial.overlap = 0
    serial.monitor_every = 0
    ref = run_case(serial, collect_fields=True)
    rep = compare_fields(ref.fields, test.fields, cfg.verify_tol)
    rep.steps = cfg.steps
    return rep


def ssspnt(size, steps, np_, seconds, s=1e-7):
    """metrics::ssspnt (src/metrics.cpp:12-19)."""
    if size <= 0 or steps <= 0 or np_ <= 0 or not seconds > 0.0:
        raise InvalidArgument("ssspnt: size, steps, np and time must be positive")
    return s * size * steps / (np_ * seconds)


# ---- host logic ---------------------------------------------------------------

def choose_dims(np_, mode):
    out = (C.c_int * 3)()
    check(lib().cav_choose_dims(np_, A.MODES.get(mode, mode), out))
    return tuple(out)


def partition(n, dims):
    p = dims[0] * dims[1] * dims[2]
    out = (C.c_int * (6 * p))()
    check(lib().cav_partition(n[0], n[1], n[2], (C.c_int * 3)(*dims), out))
    return [(tuple(out[6 * r:6 * r + 3]), tuple(out[6 * r + 3:6 * r + 6])) for r in range(p)]


def neighbors(dims, rank):
    out = (C.c_int * 6)()
    check(lib().cav_neighbors((C.c_int * 3)(*dims), rank, out))
    return tuple(out)


def center_owner(n, dims):
    node = (C.c_int * 3)()
    owner = C.c_int()
    check(lib().cav_center_owner(n[0], n[1], n[2], (C.c_int * 3)(*dims), node, C.byref(owner)))
    return tuple(node), owner.value


def grow_grid(n, np_, mode, growth_type):
    out = (C.c_int * 3)()
    check(lib().cav_grow_grid(n[0], n[1], n[2], np_, A.MODES.get(mode, mode), growth_type, out))
    return tuple(out)


def build_plan(n, rank_at, strategy):
    entries = (A.PlanEntry * 30)()
    count = C.c_int()
    check(lib().cav_build_plan(n[0], n[1], n[2], (C.c_int * 6)(*rank_at),
                               A.STRATEGIES.get(strategy, strategy), entries, 30, C.byref(count)))
    out = []
    for e in entries[:count.value]:
        out.append({"face": e.face, "neighbor": e.neighbor,
                    "vars": [(e.var[v], e.depth[v]) for v in range(e.nvars)],
                    "scalars": e.scalars, "send_tag": e.send_tag, "recv_tag": e.recv_tag})
    return out


def overlap_regions(n, rank_at):
    internal = A.Box()
    ext = (A.Box * 6)()
    count = C.c_int()
    check(lib().cav_overlap_regions(n[0], n[1], n[2], (C.c_int * 6)(*rank_at), C.byref(internal),
                                    ext, C.byref(count)))
    return internal.as_tuple(), [ext[q].as_tuple() for q in range(count.value)]


def face_box(n, face, depth, ghost=False):
    b = A.Box()
    fn = lib().cav_face_ghost_box if ghost else lib().cav_face_interior_box
    check(fn(n[0], n[1], n[2], face, depth, C.byref(b)))
    return b.as_tuple()


def repro_value(limbs70):
    arr = np.ascontiguousarray(limbs70, dtype=np.uint64)
    return lib().cav_repro_value(arr.ctypes.data_as(C.POINTER(C.c_uint64)))


# ---- op level: device tensors in the reference Field3 layout -------------------

def _fp(fields):
    return A.FieldPtrs(*[f.data_ptr() for f in fields])


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def residual_box(fields, out, X, Y, box, sp, fmad=False):
    """kernels::residual_box on 5 CUDA float64 tensors (p,u,v,w,T)."""
    L = lib(fmad)
    check(L.cav_residual_box(C.byref(_fp(fields)), C.byref(_fp(out)), X, Y,
                             C.byref(A.Box.of(*box)), C.byref(sp), _stream()), L)


def update_box(q, r, dt, X, Y, box):
    check(lib().cav_update_box(q.data_ptr(), r.data_ptr(), dt, X, Y, C.byref(A.Box.of(*box)),
                               _stream()))


def apply_boundary_conditions(fields, n, walls, fluid):
    w = (C.c_int * 6)(*[int(x) for x in walls])
    check(lib().cav_apply_boundary_conditions(C.byref(_fp(fields)), n[0], n[1], n[2], w,
                                              C.byref(fluid), _stream()))


def compute_dt(fields, n, h, fluid, cfl):
    dt = C.c_double()
    check(lib().cav_compute_dt(C.byref(_fp(fields)), n[0], n[1], n[2], h[0], h[1], h[2],
                               C.byref(fluid), cfl, C.byref(dt), _stream()))
    return dt.value


def rescale_pressure(p, n, pc):
    check(lib().cav_rescale_pressure(p.data_ptr(), n[0], n[1], n[2], pc, _stream()))


def residual_norm_partials(res, n):
    out = np.zeros(350, dtype=np.uint64)
    check(lib().cav_residual_norm_partials(C.byref(_fp(res)), n[0], n[1], n[2],
                                           out.ctypes.data_as(C.POINTER(C.c_uint64)), _stream()))
    return out.reshape(5, 70)


def copy_box_to(f, X, Y, box, out):
    check(lib().cav_copy_box_to(f.data_ptr(), X, Y, C.byref(A.Box.of(*box)), out.data_ptr(),
                                _stream()))


def copy_box_from(f, X, Y, box, buf):
    check(lib().cav_copy_box_from(f.data_ptr(), X, Y, C.byref(A.Box.of(*box)), buf.data_ptr(),
                                  _stream()))


# ---- block level ---------------------------------------------------------------

class Block:
    """One rank's device-resident block (cav_block_*). For multi-process runs
    the arenas are exchanged as CUDA IPC handles (see bench.py)."""

    def __init__(self, rank, np_, grid, dims, strategy="v3", overlap=False, fluid=None, cfl=0.4,
                 rescale=True, corrupt_exchange=False, device=0, timeout_ms=20000.0, jitter_seed=0):
        self.L = lib()
        d = A.BlockDesc()
        d.rank, d.np = rank, np_
        d.gnx, d.gny, d.gnz = grid
        for a in range(3):
            d.dims[a] = dims[a]
        d.strategy = A.STRATEGIES.get(strategy, strategy)
        d.overlap = int(overlap)
        d.fluid = fluid if fluid is not None else fluid_for_rayleigh(1e5)
        d.cfl = cfl
        d.rescale = int(rescale)
        d.corrupt_exchange = int(corrupt_exchange)
        d.device = device
        d.timeout_ms = timeout_ms
        d.jitter_seed = jitter_seed
        self.desc = d
        self.h = C.c_void_p()
        check(self.L.cav_block_create(C.byref(d), C.byref(self.h)))
        self.next_it = 1
        self.ledger = A.Ledger()
        lo, hi = partition(grid, dims)[rank]
        self.n = tuple(hi[a] - lo[a] for a in range(3))
        self.lo = lo

    def close(self):
        if self.h:
            check(self.L.cav_block_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def arena(self):
        p = C.c_void_p()
        n = C.c_size_t()
        check(self.L.cav_block_arena(self.h, C.byref(p), C.byref(n)))
        return p.value

    def arena_ipc(self):
        buf = (C.c_ubyte * 64)()
        check(self.L.cav_block_arena_ipc(self.h, buf))
        return bytes(buf)

    def connect(self, rank, ptr=None, ipc=None):
        h = (C.c_ubyte * 64).from_buffer_copy(ipc) if ipc is not None else None
        check(self.L.cav_block_connect(self.h, rank, C.c_void_p(ptr) if ptr else None, h))

    def initialize(self):
        check(self.L.cav_block_initialize(self.h))
        self.next_it = 1

    def storage_shape(self):
        return (5, self.n[2] + 4, self.n[1] + 4, self.n[0] + 4)

    def upload(self, host5):
        a = np.ascontiguousarray(host5, dtype=np.float64)
        assert a.size == int(np.prod(self.storage_shape()))
        check(self.L.cav_block_upload(self.h, a.ctypes.data_as(C.POINTER(C.c_double))))
        self.next_it = 1

    def download(self):
        out = np.zeros(self.storage_shape())
        check(self.L.cav_block_download(self.h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def run(self, n_its, check_every=10, want_norms=False):
        """March n_its iterations; returns (seconds, [(iteration, digits[5,70], linf_bits[5])])
        with this rank's exact-norm partials per check iteration."""
        cadence = max(1, check_every)
        first = self.next_it
        nchk = sum(1 for it in range(first, first + n_its)
                   if want_norms and (it == 1 or it % cadence == 0))
        W = A.NORM_WORDS
        dig = np.zeros(max(1, nchk) * W, dtype=np.uint64)
        iters = np.zeros(max(1, nchk), dtype=np.int64)
        io = A.RunIO()
        io.first_it, io.n_its, io.check_every, io.want_norms = first, n_its, cadence, int(want_norms)
        io.norm_digits = dig.ctypes.data_as(C.POINTER(C.c_uint64))
        io.check_iters = iters.ctypes.data_as(C.POINTER(C.c_longlong))
        io.ledger = self.ledger
        st = self.L.cav_block_run(self.h, C.byref(io))
        self.ledger = io.ledger
        check(st)
        self.next_it += n_its
        return io.seconds, [(int(iters[c]), dig[c * W:c * W + 350].reshape(5, 70),
                             dig[c * W + 350:c * W + 355].copy()) for c in range(io.n_checks)]

    def bench(self, n_its):
        """Times n_its iterations: (total ms, step-kernel ms per iteration,
        ms per iteration spent waiting on peers)."""
        out = (C.c_double * 3)()
        check(self.L.cav_block_bench(self.h, n_its, out))
        self.next_it += n_its
        return out[0], out[1], out[2]

    def launches_per_iteration(self):
        return self.L.cav_block_launches_per_iteration(self.h, 0)


def digits_to_value(digits70):
    """Exact value of one variable's device digits (radix-2^32 carry-save)."""
    total = 0
    for d, x in enumerate(np.asarray(digits70, dtype=np.uint64).tolist()):
        total += int(x) << (32 * d)
    # total = sum * 2^1140, round to nearest even double
    if total == 0:
        return 0.0
    return _round_scaled(total, 1140)


def _round_scaled(m, shift):
    top = m.bit_length() - 1
    if top <= 52:
        return math.ldexp(m, -shift)
    keep = m >> (top - 52)
    guard = (m >> (top - 53)) & 1
    sticky = (m & ((1 << (top - 53)) - 1)) != 0
    if guard and (sticky or (keep & 1)):
        keep += 1
        if keep == 1 << 53:
            keep >>= 1
            top += 1
    return math.ldexp(keep, top - 52 - shift)
