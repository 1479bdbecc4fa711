"""Host-side logic of the library (decomposition, plan, overlap regions, exact
sums) against tables generated from the reference (tests/golden/golden.json)
and the reference's own literal test expectations (tests/test_decomp.cpp,
tests/test_exchange.cpp, tests/test_overlap.cpp, tests/acceptance.cpp c2/c3).
No GPU needed: these entry points are plain C++ inside the .so."""
import ast

import numpy as np
import pytest

from paper_2006_02602_b200 import capi
from paper_2006_02602_b200.capi import InvalidArgument


def test_choose_dims_table(golden):
    for key, want in golden["tables"]["choose_dims"].items():
        np_, mode = (int(x) for x in key.split(","))
        if want is None:
            with pytest.raises(InvalidArgument):
                capi.choose_dims(np_, mode)
        else:
            assert list(capi.choose_dims(np_, mode)) == want, key


def test_partition_and_center_tables(golden):
    for key, want in golden["tables"]["partition"].items():
        n, dims = (ast.literal_eval(x) for x in key.split("|"))
        if want is None:
            with pytest.raises(InvalidArgument):
                capi.partition(n, dims)
            continue
        got = capi.partition(n, dims)
        flat = [x for lo, hi in got for x in (*lo, *hi)]
        assert flat == want, key
        node, owner = capi.center_owner(n, dims)
        assert list(node) + [owner] == golden["tables"]["center"][key], key


def test_grow_grid_table(golden):
    for key, want in golden["tables"]["grow"].items():
        base, np_, mode, typ = key.split("|")
        base = ast.literal_eval(base)
        if want is None:
            with pytest.raises(InvalidArgument):
                capi.grow_grid(base, int(np_), int(mode), int(typ))
        else:
            assert list(capi.grow_grid(base, int(np_), int(mode), int(typ))) == want, key


def test_paper_tables_weak_growth():
    """Paper Tables 1-2 as pinned by acceptance c3 (tests/acceptance.cpp:209-257)."""
    base = (256, 256, 256)
    assert capi.grow_grid(base, 2, "3d", 2) == (256, 256, 512)
    assert capi.grow_grid(base, 4, "3d", 2) == (256, 512, 512)
    assert capi.grow_grid(base, 8, "3d", 2) == (512, 512, 512)
    assert capi.grow_grid(base, 8, "1d-k", 2) == (256, 256, 2048)
    assert capi.grow_grid(base, 16, "3d", 2) == (512, 512, 1024)


def test_plan_table(golden):
    for key, want in golden["tables"]["plans"].items():
        n, mask, s = key.split("|")
        n = ast.literal_eval(n)
        mask, s = int(mask), int(s)
        rank_at = [100 + f if mask & (1 << f) else -1 for f in range(6)]
        got = capi.build_plan(n, rank_at, s)
        flat = [[e["face"], e["neighbor"], len(e["vars"]), [v for v, _ in e["vars"]],
                 [d for _, d in e["vars"]], e["scalars"], e["send_tag"], e["recv_tag"]] for e in got]
        assert flat == want, key


def test_plan_shapes_128_cube():
    """tests/test_exchange.cpp:47-91 incl. the exact 6/10 ratio (acceptance c2)."""
    n = (128, 128, 128)
    t = [1, 2, 3, 4, 5, 6]
    area = 128 * 128
    base = capi.build_plan(n, t, "baseline")
    assert len(base) == 30 and all(e["scalars"] == 2 * area for e in base)
    v1 = capi.build_plan(n, t, "v1")
    assert len(v1) == 22 and sum(e["scalars"] for e in v1) == 30 * 2 * area
    v2 = capi.build_plan(n, t, "v2")
    ilow1 = [e for e in v1 if e["face"] == 0][0]
    ilow2 = [e for e in v2 if e["face"] == 0][0]
    assert ilow2["scalars"] == 6 * area and ilow2["scalars"] * 10 == ilow1["scalars"] * 6
    v3 = capi.build_plan(n, t, "v3")
    assert len(v3) == 6
    for e in v3:
        assert e["scalars"] == 6 * area
        assert [d for v, d in e["vars"]] == [2, 1, 1, 1, 1]
        assert e["recv_tag"] == e["face"] * 8 and e["send_tag"] == (e["face"] ^ 1) * 8


def test_overlap_regions_table(golden):
    for key, want in golden["tables"]["overlap"].items():
        n, mask = key.split("|")
        n = ast.literal_eval(n)
        mask = int(mask)
        rank_at = [100 + f if mask & (1 << f) else -1 for f in range(6)]
        internal, ext = capi.overlap_regions(n, rank_at)
        got = [[list(internal[0]), list(internal[1])]] + [[list(b[0]), list(b[1])] for b in ext]
        assert got == [[list(b[0]), list(b[1])] for b in want], key


def test_overlap_cover_all_topologies():
    """tests/test_overlap.cpp:61-103: disjoint cover, halo-dependent cells external."""
    n = (8, 9, 10)
    for mask in range(64):
        rank_at = [100 + f if mask & (1 << f) else -1 for f in range(6)]
        internal, ext = capi.overlap_regions(n, rank_at)
        paint = np.zeros((n[2] + 4, n[1] + 4, n[0] + 4), dtype=int)
        (lo, hi) = internal
        paint[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] += 1
        for lo, hi in ext:
            paint[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] += 2
        inner = paint[2:-2, 2:-2, 2:-2]
        assert set(np.unique(inner)) <= {1, 2}
        for f in range(6):
            if mask & (1 << f):
                a, side = f // 2, f % 2
                sl = [slice(None)] * 3
                ax = 2 - a
                sl[ax] = slice(0, 2) if side == 0 else slice(-2, None)
                assert np.all(inner[tuple(sl)] == 2)


def test_face_boxes():
    n = (7, 6, 5)
    assert capi.face_box(n, 0, 2) == ((2, 2, 2), (4, 8, 7))
    assert capi.face_box(n, 1, 1, ghost=True) == ((9, 2, 2), (10, 8, 7))
    assert capi.face_box(n, 4, 2, ghost=True) == ((2, 2, 0), (9, 8, 2))
    with pytest.raises(InvalidArgument, match="depth must be 1..2"):
        capi.face_box(n, 0, 3)


def test_repro_value_rounding():
    """ReproSum::value rounding (inc/util/repro_sum.hpp:48-77): ties to even."""
    limbs = np.zeros(70, dtype=np.uint64)
    # value*2^1140 = 2^53 + 1 (a tie at 2^53 scale) -> rounds to even 2^53
    limbs[0] = (1 << 53) + 1
    assert capi.repro_value(limbs) == np.ldexp(2.0 ** 53, -1140)
    limbs[0] = (1 << 53) + 3  # tie, odd keep -> rounds up
    assert capi.repro_value(limbs) == np.ldexp(2.0 ** 53 + 4, -1140)
    limbs[0] = 0
    limbs[20] = 1  # 2^1280 * 2^-1140 = 2^140
    assert capi.repro_value(limbs) == 2.0 ** 140
    limbs[35 + 20] = 1  # negative half equal: exact zero
    assert capi.repro_value(limbs) == 0.0


def test_digits_value_matches_limbs():
    rng = np.random.default_rng(3)
    dig = rng.integers(0, 2 ** 40, 70, dtype=np.uint64)
    dig[60:] = 0
    total = sum(int(x) << (32 * d) for d, x in enumerate(dig.tolist()))
    limbs = np.array([(total >> (64 * l)) & (2 ** 64 - 1) for l in range(35)] + [0] * 35,
                     dtype=np.uint64)
    assert capi.digits_to_value(dig) == capi.repro_value(limbs)


def test_config_defaults_match_reference():
    """RunConfig/SolverConfig/FluidParams defaults (inc/util/config.hpp:15-34)."""
    from oracle.refbind import Ref, ref_available
    cfg = capi.default_config()
    assert (cfg.nx, cfg.ny, cfg.nz, cfg.np, cfg.steps) == (32, 32, 32, 1, -1)
    assert cfg.cfl == 0.4 and cfg.check_every == 10 and cfg.conv_tol == 1e-8
    assert cfg.max_steps == 200000 and cfg.rescale == 1 and cfg.verify_tol == 1e-12
    if ref_available():
        import ctypes as C
        from paper_2006_02602_b200 import _abi as A
        ref = A.RunConfig()
        Ref.lib().ref_run_config_default(C.byref(ref))
        assert bytes(ref.fluid) == bytes(cfg.fluid)
        for f in ("nx", "np", "mode", "strategy", "steps", "cfl", "max_steps", "conv_tol",
                  "rescale", "check_every", "timeout_ms", "verify_tol"):
            assert getattr(ref, f) == getattr(cfg, f), f


def test_validation_messages():
    with pytest.raises(InvalidArgument, match="choose_dims: 2d cannot split a prime rank count 7"):
        capi.choose_dims(7, "2d")
    with pytest.raises(InvalidArgument, match="gives 4-node blocks; minimum is 5"):
        capi.partition((8, 8, 8), (2, 1, 1))
    with pytest.raises(InvalidArgument, match="np must be a power of two, got 3"):
        capi.grow_grid((32, 32, 32), 3, "3d", 2)
    with pytest.raises(InvalidArgument, match="grid: axis j has 4 nodes, minimum is 5"):
        capi.cavity_spacing((8, 4, 8))
