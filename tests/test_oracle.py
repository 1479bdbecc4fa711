"""The plain-C oracle (oracle/cavity_oracle.c) pinned against fixtures generated
from the reference itself (tests/golden/make_golden.py), and — where the
reference library was built (oracle/_ref) — against the reference directly."""
import ctypes as C
import hashlib

import numpy as np
import pytest

from conftest import golden_config
from oracle.refbind import CheckerError, Oracle, Ref, default_config, ref_available
from paper_2006_02602_b200 import _abi as A


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def oracle_residual(f, n, h, box):
    L = Oracle.lib()
    sp = A.StencilParams()
    L.oc_make_stencil_params(C.c_double(h[0]), C.c_double(h[1]), C.c_double(h[2]),
                             C.byref(default_config().fluid), C.byref(sp))
    out = np.zeros_like(f)
    fp = A.FieldPtrs(*[f[v].ctypes.data for v in range(5)])
    op = A.FieldPtrs(*[out[v].ctypes.data for v in range(5)])
    L.oc_residual_box(C.byref(fp), C.byref(op), n[0] + 4, n[1] + 4, C.byref(A.Box.of(*box)),
                      C.byref(sp))
    return out


@pytest.mark.parametrize("nx", [5, 9, 12])
def test_oracle_residual_matches_reference_golden(golden_arrays, nx):
    g = golden_arrays["residual"]
    n = (nx, 7, 6)
    box = ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2))
    out = oracle_residual(g[f"in_{nx}"], n, tuple(g[f"h_{nx}"]), box)
    np.testing.assert_array_equal(bits(out), bits(g[f"out_{nx}"]))


@pytest.mark.parametrize("name", ["c0_32_1000", "r16x12x9_200", "r10_50_norescale",
                                  "r12_60_cfl07_every7", "conv16_max300", "quiescent_conv",
                                  "ra1e4_20x16x12_120"])
def test_oracle_run_matches_reference_golden(golden, golden_arrays, name):
    entry = golden["runs"][name]
    cfg = golden_config(entry, default_config)
    r = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    assert r["steps_marched"] == entry["steps_marched"]
    assert r["converged"] == entry["converged"]
    assert [int(x) for x in r["history_iter"]] == entry["history_iter"]
    want = np.array([[float.fromhex(x) for x in row] for row in entry["history"]])
    np.testing.assert_array_equal(bits(r["history"]), bits(want))
    assert [sha(r["fields"][v]) for v in range(5)] == entry["fields_sha256"]
    if name in golden_arrays["runs"]:
        np.testing.assert_array_equal(bits(r["fields"]), bits(golden_arrays["runs"][name]))


def test_oracle_c0_fingerprints(golden):
    """SURVEY §8c fingerprints of C0 (32^3, 1000 steps): norms at it=1000."""
    h = golden["runs"]["c0_32_1000"]["history"]
    assert len(h) == 101
    assert float.fromhex(h[-1][0]) == 2.0448558943954212e-05
    assert float.fromhex(h[0][4]) == 2.0302816901408454


@pytest.mark.parametrize("name", ["diverge_cfl50", "diverge_cfl50_every1", "diverge_12cube",
                                  "bad_cfl"])
def test_oracle_error_paths_match_reference(golden, name):
    e = golden["errors"][name]
    kw = dict(e["config"])
    kw["grid"] = tuple(kw["grid"])
    with pytest.raises(CheckerError) as ex:
        Oracle.run_case(default_config(**kw), collect_history=e["history"])
    assert str(ex.value) == e["error"]


def test_oracle_repro_value_rounding():
    """ReproSum::value rounding (inc/util/repro_sum.hpp:48-77), restated."""
    L = Oracle.lib()

    def val(limbs):
        arr = np.ascontiguousarray(limbs, dtype=np.uint64)
        return L.oc_repro_value(arr.ctypes.data_as(C.POINTER(C.c_uint64)))

    limbs = np.zeros(70, dtype=np.uint64)
    limbs[0] = (1 << 53) + 1  # tie -> even
    assert val(limbs) == np.ldexp(2.0 ** 53, -1140)
    limbs[0] = (1 << 53) + 3  # tie, odd keep -> up
    assert val(limbs) == np.ldexp(2.0 ** 53 + 4, -1140)
    limbs[:] = 0
    limbs[35] = 5  # negative half only
    assert val(limbs) == -np.ldexp(5.0, -1140)


@pytest.mark.skipif(not ref_available(), reason="reference library not built here")
def test_oracle_norm_partials_equal_reference_limbs():
    """Exact partials (serialised ReproSum limbs) equal the reference's."""
    import oracle_ops as O
    n = (9, 7, 6)
    r = O.random_fields(n, 5)
    r[2] *= 1e-158
    want = np.zeros(350, dtype=np.uint64)
    fp = A.FieldPtrs(*[r[v].ctypes.data for v in range(5)])
    assert Ref.lib().ref_residual_norm_partials(C.byref(fp), n[0], n[1], n[2],
                                                want.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    np.testing.assert_array_equal(O.norm_limbs(r, n).ravel(), want)


@pytest.mark.skipif(not ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("kw", [dict(grid=(14, 11, 9), steps=40), dict(grid=(9, 9, 13), steps=30,
                                                                      check_every=3)])
def test_oracle_vs_reference_live(kw):
    cfg = default_config(**kw)
    a = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    b = Ref.run_case(cfg, collect_fields=True, collect_history=True)
    np.testing.assert_array_equal(bits(a["fields"]), bits(b["fields"]))
    np.testing.assert_array_equal(bits(a["history"]), bits(b["history"]))
