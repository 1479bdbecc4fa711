"""run_case on the GPU vs the reference, bitwise (tests/test_runner.cpp,
tests/acceptance.cpp c1/c6/c7/c8 analogues). Multi-rank cases put every rank
on device 0 — the in-process block group is the same code path as one rank
per GPU, with peer pointers on the same device."""
import hashlib

import numpy as np
import pytest

import oracle_ops as O
from conftest import golden_config
from oracle.refbind import Oracle
from paper_2006_02602_b200 import _abi, capi
from paper_2006_02602_b200.capi import CavityError, InvalidArgument

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


GOLDEN_RUNS = ["c0_32_1000", "r16x12x9_200", "r10_50_norescale", "r12_60_cfl07_every7",
               "conv16_max300", "quiescent_conv", "ra1e4_20x16x12_120"]


def check_against_golden(r, entry, golden_arrays, name):
    assert r.steps_marched == entry["steps_marched"]
    assert r.converged == entry["converged"]
    assert [int(x) for x in r.history_iter] == entry["history_iter"]
    want = np.array([[float.fromhex(x) for x in row] for row in entry["history"]])
    np.testing.assert_array_equal(bits(r.history), bits(want))
    if name in golden_arrays["runs"]:
        np.testing.assert_array_equal(bits(r.fields), bits(golden_arrays["runs"][name]))
    assert [sha(r.fields[v]) for v in range(5)] == entry["fields_sha256"]


@pytest.mark.parametrize("name", GOLDEN_RUNS)
def test_serial_run_matches_reference(golden, golden_arrays, name):
    entry = golden["runs"][name]
    cfg = golden_config(entry, capi.default_config)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    check_against_golden(r, entry, golden_arrays, name)


@pytest.mark.parametrize("np_,mode,strategy,overlap", [
    (8, "3d", "v3", 1), (8, "3d", "baseline", 0), (4, "1d-i", "v2", 1), (4, "2d", "v1", 0),
    (2, "1d-k", "v3", 1), (6, "3d", "v3", 1)])
def test_parallel_c0_matches_reference(golden, golden_arrays, np_, mode, strategy, overlap):
    """C0 (32^3, 1000 steps) decomposed: fields and history bitwise equal to
    the reference's serial run (acceptance c1/c7)."""
    entry = golden["runs"]["c0_32_1000"]
    cfg = golden_config(entry, capi.default_config)
    _abi.apply_overrides(cfg, np=np_, mode=mode, strategy=strategy, overlap=overlap)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    check_against_golden(r, entry, golden_arrays, "c0_32_1000")
    assert r.np == np_


@pytest.mark.parametrize("strategy", ["baseline", "v1", "v2", "v3"])
@pytest.mark.parametrize("mode", ["1d-i", "2d", "3d"])
@pytest.mark.parametrize("overlap", [0, 1])
def test_every_strategy_and_mode_agrees_with_serial(strategy, mode, overlap):
    """tests/test_runner.cpp:54-72 (+ overlap)."""
    cfg = capi.default_config(grid=(20, 16, 16), steps=10, np=4, mode=mode, strategy=strategy,
                              overlap=overlap)
    r = capi.run_case(cfg, collect_fields=True)
    o = Oracle.run_case(capi.default_config(grid=(20, 16, 16), steps=10), collect_fields=True)
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    rep = capi.verify_against_serial(cfg)
    assert rep.passed and all(d == 0.0 for d in rep.max_abs)


def test_ragged_partition_np6_and_np12():
    for np_, mode, grid in [(6, "3d", (23, 17, 29)), (12, "3d", (31, 26, 21)), (3, "1d-j", (9, 17, 8))]:
        cfg = capi.default_config(grid=grid, steps=15, np=np_, mode=mode, overlap=1)
        r = capi.run_case(cfg, collect_fields=True, collect_history=True)
        o = Oracle.run_case(capi.default_config(grid=grid, steps=15), collect_fields=True,
                            collect_history=True)
        np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
        np.testing.assert_array_equal(bits(r.history), bits(o["history"]))


def test_corrupted_halo_fails_verification():
    """tests/test_runner.cpp:87-102: the negative control must FAIL."""
    cfg = capi.default_config(grid=(16, 16, 16), steps=10, np=4)
    clean = capi.verify_against_serial(cfg)
    assert clean.passed and "PASS" in clean.summary()
    bad = capi.verify_against_serial(cfg, corrupt_exchange=True)
    assert not bad.passed and max(bad.max_abs) > 0.0 and "FAIL" in bad.summary()


@pytest.mark.parametrize("name", ["diverge_cfl50", "diverge_cfl50_every1", "diverge_12cube",
                                  "bad_cfl", "diverge_cfl50_np2", "diverge_cfl50_every1_np2",
                                  "diverge_12cube_np2", "bad_cfl_np2"])
def test_error_paths_match_reference(golden, name):
    """'iteration N: ...' wrapping (src/runner.cpp:231-233), the norms-first
    order on check iterations, and the root cause across ranks."""
    e = golden["errors"][name]
    kw = dict(e["config"])
    kw["grid"] = tuple(kw["grid"])
    with pytest.raises(CavityError) as ex:
        capi.run_case(capi.default_config(**kw), collect_history=e["history"])
    assert str(ex.value) == e["error"]


def test_history_cadence():
    cfg = capi.default_config(grid=(16, 16, 16), steps=25, check_every=10)
    r = capi.run_case(cfg, collect_history=True)
    assert list(r.history_iter) == [1, 10, 20]
    assert np.all(np.isfinite(r.history))
    assert len(capi.run_case(cfg).history) == 0


def test_ledger_totals():
    """tests/test_runner.cpp:162-179."""
    cfg = capi.default_config(grid=(16, 16, 16), steps=5, np=2, mode="1d-k", strategy="v3")
    r = capi.run_case(cfg)
    per_exchange = 6 * 16 * 16 * 8
    for led in r.ledgers:
        assert led["exchanges"] == 5
        assert led["messages_sent"] == 5
        assert led["bytes_sent"] == 5 * per_exchange
    assert r.bytes_sent == 2 * 5 * per_exchange


def test_zero_steps_returns_initial_condition():
    cfg = capi.default_config(grid=(16, 16, 16), steps=0, np=2)
    r = capi.run_case(cfg, collect_fields=True)
    assert r.steps_marched == 0 and r.steps_timed == 0 and np.isnan(r.ssspnt)
    assert np.all(r.fields[:4] == 0.0) and np.all(r.fields[4] == cfg.fluid.t_inf)


def test_quiescent_converges_immediately_parallel():
    for np_ in (1, 4):
        cfg = capi.default_config(grid=(16, 16, 16), steps=-1, t_hot=300.0, t_cold=300.0, np=np_)
        r = capi.run_case(cfg)
        assert r.converged and r.steps_marched == 1


def test_bad_configurations():
    with pytest.raises(InvalidArgument):
        capi.run_case(capi.default_config(grid=(16, 16, 16), steps=5, np=0))
    with pytest.raises(InvalidArgument):
        capi.run_case(capi.default_config(grid=(16, 16, 16), steps=5, np=513))
    with pytest.raises(InvalidArgument):
        capi.verify_against_serial(capi.default_config(grid=(16, 16, 16), steps=-1, np=2))
    with pytest.raises(InvalidArgument):
        capi.run_case(capi.default_config(grid=(16, 16, 16), steps=5, nu=-1.0))
    with pytest.raises(InvalidArgument, match="minimum is 5"):
        capi.run_case(capi.default_config(grid=(16, 16, 8), steps=5, np=2, mode="1d-k"))


def test_record_fields():
    cfg = capi.default_config(grid=(16, 16, 16), steps=30, np=8, strategy="v3", overlap=1)
    r = capi.run_case(cfg)
    assert r.steps_marched == 30 and r.steps_timed == 29 and not r.converged
    assert r.np == 8 and r.dims == (2, 2, 2)
    assert r.wall_time_s > 0 and r.bytes_sent > 0
    assert r.ssspnt == pytest.approx(capi.ssspnt(16 ** 3, 29, 8, r.wall_time_s))


def test_block_api_from_arbitrary_state():
    """Block upload -> run -> download equals the oracle's loop on the same
    state, including every ghost cell (lazy rescale undone exactly)."""
    n = (21, 10, 13)
    f = O.random_fields(n, 99, vel=0.02)
    f[0] *= 1e-3
    b = capi.Block(0, 1, n, (1, 1, 1))
    b.upload(f)
    b.run(3)
    got = b.download()
    h = capi.cavity_spacing(n)
    want = O.march(f, n, h, capi.fluid_for_rayleigh(1e5), 0.4, 3)
    np.testing.assert_array_equal(bits(got), bits(want))
    b.run(2)
    want = O.march(want, n, h, capi.fluid_for_rayleigh(1e5), 0.4, 2)
    np.testing.assert_array_equal(bits(b.download()), bits(want))
    b.close()


def test_fused_step_large_block_matches_oracle():
    """The tiled fused kernel on a block larger than one tile in every axis,
    with ragged edges, vs the oracle loop."""
    n = (70, 37, 45)
    cfg = capi.default_config(grid=n, steps=12)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    o = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))


@pytest.mark.parametrize("name", ["r16x12x9_200", "ra1e4_20x16x12_120"])
def test_fmad_tolerance_build_within_1e10(golden, golden_arrays, name):
    """The FMA-contracted build (libcavity_b200_fmad.so) is not bitwise, but
    stays within BASELINE.json's 1e-10 relative tolerance (compare_fields
    metric, src/runner.cpp:355-375) on fields and the norm history."""
    entry = golden["runs"][name]
    cfg = golden_config(entry, capi.default_config)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True, fmad=True)
    rep = capi.compare_fields(golden_arrays["runs"][name], r.fields, 1e-10)
    assert rep.passed, rep.summary()
    want = np.array([[float.fromhex(x) for x in row] for row in entry["history"]])
    rel = np.abs(r.history - want) / np.maximum(np.abs(want), 1e-300)
    assert np.all(rel[want != 0] <= 1e-10)


# ---- BASELINE.json configs[1] at its full size (256^3) -----------------------

C1 = (256, 256, 256)


def test_c1_full_size_matches_oracle_bitwise():
    """configs[1]'s grid, a few iterations with the residual-norm history at
    every step: fields and norms bitwise equal to the C oracle (which is itself
    pinned to the reference, tests/test_oracle.py). Exercises the production
    TMA step at its benchmark size: all tile classes, dynamic items, tail
    chunks, eager rescale and the last-CTA fold."""
    cfg = capi.default_config(grid=C1, steps=5, check_every=1)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    o = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    assert list(r.history_iter) == list(o["history_iter"])
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))


@pytest.mark.parametrize("np_, mode, overlap", [(2, "1d-i", 1), (8, "3d", 1), (4, "2d", 0)])
def test_c1_full_size_decomposition_independent(np_, mode, overlap):
    """Size-independent property at full size: the reference is bitwise
    independent of decomposition (P/README.md:10-15), so every rank layout of
    the 256^3 case reproduces the single-rank fields and norms bit for bit
    (ranks share device 0 here; the halo exchange, lazy rescale and scalar
    sync are the multi-GPU code path)."""
    base = capi.default_config(grid=C1, steps=4, check_every=2)
    one = capi.run_case(base, collect_fields=True, collect_history=True)
    many = capi.run_case(capi.default_config(grid=C1, steps=4, check_every=2, np=np_, mode=mode, strategy="v3",
                                             overlap=overlap), collect_fields=True, collect_history=True)
    np.testing.assert_array_equal(bits(many.fields), bits(one.fields))
    np.testing.assert_array_equal(bits(many.history), bits(one.history))


@pytest.mark.parametrize("u_ref, np_", [(1e-3, 1), (0.02, 1), (1e-3, 2)])
def test_beta_branches_match_oracle(u_ref, np_):
    """beta = max(|V|, u_ref) (compute_beta): with u_ref below the flow speed
    (max|V| ~ 0.036 here) the step kernel's exact shortcuts are bypassed —
    the high-word test fails and s2 exceeds beta_fast_s2 — so the IEEE sqrt
    branch, the mixed warps and the CFL maxima over sqrt-derived betas are
    all exercised; u_ref = 0.02 mixes cells on both sides of u_ref/2 and u_ref.
    Bitwise vs the oracle, fields and norm history."""
    kw = dict(grid=(24, 20, 16), steps=80, check_every=5, u_ref=u_ref)
    if np_ > 1:
        kw.update(np=np_, mode="1d-i", strategy="v3", overlap=1)
    r = capi.run_case(capi.default_config(**kw), collect_fields=True, collect_history=True)
    o = Oracle.run_case(capi.default_config(grid=(24, 20, 16), steps=80, check_every=5, u_ref=u_ref),
                        collect_fields=True, collect_history=True)
    assert np.abs(o["fields"].reshape(5, -1)[1:4]).max() > u_ref  # the flow does outrun u_ref
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))


def test_c0_solve_to_convergence_matches_oracle():
    """`cavity solve`'s default mode on configs[0]'s grid: march until the
    convergence rule holds (src/runner.cpp:210-220), decided on the device
    after every check, no host round trip per check. Same converged
    iteration (~6600, P/README.md:43-44), fields and norm history as the
    oracle, bitwise."""
    cfg = capi.default_config(grid=(32, 32, 32), steps=-1)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    o = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    assert r.converged and o["converged"]
    assert r.steps_marched == o["steps_marched"]
    assert list(r.history_iter) == list(o["history_iter"])
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))


@pytest.mark.parametrize("env", [{"CAV_STORED_GHOSTS": "1"}, {"CAV_STORED_GHOSTS": "1", "CAV_GHOST_WRITES": "0"},
                                 {"CAV_STORED_GHOSTS": "0"}])
@pytest.mark.parametrize("n", [(67, 19, 11), (33, 9, 7), (34, 12, 5), (64, 8, 6)])
def test_stored_wall_ghosts_match_oracle(monkeypatch, env, n):
    """Single-rank steps with the wall ghosts stored in the state (x walls by
    the step kernel's wall lanes when three interior layers share a warp, the
    rest by k_bc), with k_bc only, and with register ghosts: all bitwise equal
    to the oracle, ghost cells included (block API, arbitrary state)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    f = O.random_fields(n, 7 + n[0], vel=0.03)
    f[0] *= 1e-3
    b = capi.Block(0, 1, n, (1, 1, 1))
    b.upload(f)
    b.run(5)
    h = capi.cavity_spacing(n)
    want = O.march(f, n, h, capi.fluid_for_rayleigh(1e5), 0.4, 5)
    np.testing.assert_array_equal(bits(b.download()), bits(want))
    b.run(2)
    want = O.march(want, n, h, capi.fluid_for_rayleigh(1e5), 0.4, 2)
    np.testing.assert_array_equal(bits(b.download()), bits(want))
    b.close()


@pytest.mark.parametrize("grid", [(24, 20, 16), (37, 21, 13)])
def test_stored_ghosts_norm_history_matches_oracle(monkeypatch, grid):
    """The stored-ghost step (forced on below its size threshold) with norm
    iterations every 5th step and a developed flow: fields and the residual
    norm history bitwise equal to the oracle."""
    monkeypatch.setenv("CAV_STORED_GHOSTS", "1")
    cfg = capi.default_config(grid=grid, steps=80, check_every=5, u_ref=1e-3)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    o = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))
