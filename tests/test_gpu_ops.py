"""Op-level sm_100a kernels vs the CPU oracle, bitwise (the reference's
backend-equivalence tests, tests/test_kernels.cpp:77-167 and
tests/test_solver.cpp, with the Cuda backend in place of AVX2)."""
import numpy as np
import pytest

import oracle_ops as O
from paper_2006_02602_b200 import capi
from paper_2006_02602_b200.capi import InvalidArgument, CavityError

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def fluid():
    return capi.fluid_for_rayleigh(1e5)


@pytest.mark.parametrize("nx", [5, 9, 12])
def test_residual_matches_reference_golden(golden_arrays, nx):
    g = golden_arrays["residual"]
    n = (nx, 7, 6)
    h = tuple(g[f"h_{nx}"])
    sp = capi.stencil_params(*h, fluid())
    fin = [dev(g[f"in_{nx}"][v]) for v in range(5)]
    out = [torch.zeros_like(x) for x in fin]
    capi.residual_box(fin, out, n[0] + 4, n[1] + 4, ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2)), sp)
    got = np.stack([host(t) for t in out])
    np.testing.assert_array_equal(bits(got), bits(g[f"out_{nx}"]))


@pytest.mark.parametrize("box", [((2, 2, 2), (3, 12, 11)), ((3, 4, 5), (18, 5, 6)),
                                 ((5, 3, 4), (11, 9, 8)), ((2, 2, 2), (18, 12, 11))])
def test_residual_sub_boxes(box):
    n = (16, 10, 9)
    f = O.random_fields(n, 77)
    h = (0.05 / 15, 0.06 / 9, 0.045 / 8)
    sp = capi.stencil_params(*h, fluid())
    want = O.residual(f, n, box, O.stencil(h, fluid()))
    fin = [dev(f[v]) for v in range(5)]
    out = [torch.zeros_like(x) for x in fin]
    capi.residual_box(fin, out, n[0] + 4, n[1] + 4, box, sp)
    got = np.stack([host(t) for t in out])
    np.testing.assert_array_equal(bits(got), bits(want))


@pytest.mark.parametrize("nx", [5, 9, 13])
def test_update_box(nx):
    n = (nx, 6, 5)
    f = O.random_fields(n, 31 + nx)
    box = ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2))
    want = O.update(f[0], f[4], 1.7e-3, n, box)
    q = dev(f[0])
    capi.update_box(q, dev(f[4]), 1.7e-3, n[0] + 4, n[1] + 4, box)
    np.testing.assert_array_equal(bits(host(q)), bits(want))


@pytest.mark.parametrize("walls", [(1, 1, 1, 1, 1, 1), (1, 0, 1, 1, 0, 1), (0, 0, 0, 0, 0, 1)])
def test_boundary_conditions(walls):
    n = (6, 7, 8)
    f = O.random_fields(n, 2024)
    want = O.bc(f, n, walls, fluid())
    t = [dev(f[v]) for v in range(5)]
    capi.apply_boundary_conditions(t, n, walls, fluid())
    got = np.stack([host(x) for x in t])
    np.testing.assert_array_equal(bits(got), bits(want))


def test_compute_dt_closed_form_and_random():
    n = (32, 32, 32)
    fl = fluid()
    h = capi.cavity_spacing(n)
    f = np.zeros((5, 36, 36, 36))
    f[4] = fl.t_inf
    t = [dev(f[v]) for v in range(5)]
    conv = h[0] / fl.u_ref
    visc = h[0] * h[0] / (6.0 * fl.nu)
    therm = h[0] * h[0] / (6.0 * fl.alpha)
    assert capi.compute_dt(t, n, h, fl, 0.4) == 0.4 * min(conv, visc, therm)
    g = O.random_fields((9, 8, 7), 5, vel=2.0)
    t = [dev(g[v]) for v in range(5)]
    hh = (0.01, 0.012, 0.009)
    assert capi.compute_dt(t, (9, 8, 7), hh, fl, 0.7) == O.compute_dt(g, (9, 8, 7), hh, fl, 0.7)


def test_compute_dt_errors():
    n = (6, 6, 6)
    fl = fluid()
    f = np.zeros((5, 10, 10, 10))
    f[4] = fl.t_inf
    f[3][5, 5, 5] = np.nan
    t = [dev(f[v]) for v in range(5)]
    with pytest.raises(InvalidArgument):
        capi.compute_dt(t, n, (0.01,) * 3, fl, 0.0)
    with pytest.raises(CavityError, match="non-finite value in field w"):
        capi.compute_dt(t, n, (0.01,) * 3, fl, 0.4)
    f[0][3, 3, 3] = np.inf  # p is scanned first (P,U,V,W,T order)
    t = [dev(f[v]) for v in range(5)]
    with pytest.raises(CavityError, match="non-finite value in field p$"):
        capi.compute_dt(t, n, (0.01,) * 3, fl, 0.4)


def test_rescale():
    n = (6, 6, 6)
    f = O.random_fields(n, 9)
    pc = f[0][4, 4, 4]
    p = dev(f[0])
    capi.rescale_pressure(p, n, pc)
    np.testing.assert_array_equal(bits(host(p)), bits(O.rescale(f[0], n, pc)))


@pytest.mark.parametrize("n,seed", [((6, 6, 6), 31), ((17, 9, 11), 4), ((40, 33, 21), 8)])
def test_norm_partials_exact(n, seed):
    r = O.random_fields(n, seed)
    r[2] *= 1e-158  # squares land in the subnormal range
    r[3][2, 2, 2] = 0.0
    want = O.norm_limbs(r, n)
    got = capi.residual_norm_partials([dev(r[v]) for v in range(5)], n)
    np.testing.assert_array_equal(got, want)
    for v in range(5):
        assert capi.repro_value(got[v]) == capi.repro_value(want[v])


def test_norm_partials_non_finite():
    n = (6, 6, 6)
    r = O.random_fields(n, 1)
    r[1][3, 3, 3] = 1e300  # square overflows: "repro_sum: non-finite term"
    with pytest.raises(InvalidArgument, match="repro_sum: non-finite term"):
        capi.residual_norm_partials([dev(r[v]) for v in range(5)], n)


@pytest.mark.parametrize("face", range(6))
@pytest.mark.parametrize("depth", [1, 2])
def test_copy_box_index_maps(face, depth):
    """Pack/unpack index maps bit-exact (src/slab.cpp:51-71)."""
    n = (7, 6, 5)
    f = O.random_fields(n, face * 7 + depth)[0]
    for ghost in (False, True):
        box = capi.face_box(n, face, depth, ghost)
        want = O.copy_box_to(f, n, box)
        buf = torch.zeros(want.size, dtype=torch.float64, device="cuda")
        capi.copy_box_to(dev(f), n[0] + 4, n[1] + 4, box, buf)
        np.testing.assert_array_equal(bits(host(buf)), bits(want))
        g = dev(np.zeros_like(f))
        capi.copy_box_from(g, n[0] + 4, n[1] + 4, box, dev(want))
        back = host(g)
        lo, hi = box
        np.testing.assert_array_equal(back[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]],
                                      f[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]])


@pytest.mark.parametrize("box", [((2, 2, 2), (2, 12, 11)), ((5, 3, 4), (11, 3, 8)), ((4, 4, 4), (3, 9, 9))])
def test_empty_boxes_are_no_ops(box):
    """residual_box / update_box on an empty box (some hi <= lo) write
    nothing, as the reference's loops do (src/kernels_scalar.cpp:5-30)."""
    n = (16, 10, 9)
    f = O.random_fields(n, 5)
    h = (0.05 / 15, 0.06 / 9, 0.045 / 8)
    sp = capi.stencil_params(*h, fluid())
    fin = [dev(f[v]) for v in range(5)]
    out = [torch.full_like(x, 12345.0) for x in fin]
    capi.residual_box(fin, out, n[0] + 4, n[1] + 4, box, sp)
    assert all(bool((t == 12345.0).all()) for t in out)
    q = dev(f[1])
    capi.update_box(q, out[1], 0.25, n[0] + 4, n[1] + 4, box)
    np.testing.assert_array_equal(bits(host(q)), bits(f[1]))
