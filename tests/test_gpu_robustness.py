"""Robustness parity on the GPU path and the L-inf residual
norm north_star asks for:

* a peer that never runs raises TransportTimeout naming the waiting rank and
  every stuck (source, tag) pair, as InprocTransport::wait_all does
  (/root/reference/proj/src/inproc.cpp:145-177, pinned by
  tests/test_transport.cpp:114-133) — the waits are stream-ordered, so the
  timeout is raised by the host, and the block's streams drain afterwards;
* seeded randomized rank timing (the GPU analogue of the reference's shuffled
  delivery, src/inproc.cpp:92-114 / acceptance c8, tests/acceptance.cpp:
  591-628): two 8-rank overlapped runs with skewed rank start times and
  random pauses give byte-identical fields, norms and ledgers, equal to the
  unperturbed run;
* L-inf norms max |R_v| per check iteration equal numpy's max over the
  oracle's residual fields (the reference has only L2; src/solver.cpp:259-285
  defines which residual a check iteration reduces);
* a device-converged solve on the stored-ghost path stops where the oracle
  does, with one exchange per marched iteration in the ledger.
"""
import numpy as np
import pytest

import oracle_ops as O
from oracle.refbind import Oracle
from paper_2006_02602_b200 import capi
from paper_2006_02602_b200.capi import TransportTimeout

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_timeout_names_waiting_rank_and_stuck_sources():
    grid, dims = (30, 12, 10), (3, 1, 1)
    blocks = [capi.Block(r, 3, grid, dims, strategy="v3", timeout_ms=300.0) for r in range(3)]
    for b in blocks:
        for r in range(3):
            if r != b.desc.rank:
                b.connect(r, ptr=blocks[r].arena())
        b.initialize()
    # ranks 1 and 2 never march: rank 0 waits for their scalars and rank 1's halo
    with pytest.raises(TransportTimeout) as ex:
        blocks[0].run(3)
    msg = str(ex.value)
    assert msg.startswith("rank 0: receive timed out")
    assert "(src=1, tag=1001)" in msg and "(src=2, tag=1001)" in msg
    entry = [e for e in capi.build_plan(blocks[0].n, capi.neighbors(dims, 0), "v3")][0]
    assert f"(src=1, tag={entry['recv_tag']})" in msg
    # the aborted block refuses further work and still closes (its streams drained)
    with pytest.raises(capi.LogicError):
        blocks[0].run(1)
    for b in blocks:
        b.close()


@pytest.mark.parametrize("fused", [True, False])
def test_timeout_at_a_later_iteration(monkeypatch, fused):
    """A peer that stops after some iterations: the waiting rank names it at
    the first iteration it cannot complete. With fused halos (default) the
    peer's step n already sent S_n's halos, so iteration 5 completes and the
    wait for its scalars of iteration 5 times out at 6; the slab exchange
    (CAV_FUSED_HALO=0) sends S_4's halos at iteration 5, like the reference."""
    monkeypatch.setenv("CAV_FUSED_HALO", "1" if fused else "0")
    grid, dims = (20, 12, 10), (2, 1, 1)
    a, b = (capi.Block(r, 2, grid, dims, strategy="v3", overlap=True, timeout_ms=300.0) for r in range(2))
    a.connect(1, ptr=b.arena())
    b.connect(0, ptr=a.arena())
    a.initialize()
    b.initialize()
    import threading
    t = threading.Thread(target=lambda: b.run(4))
    t.start()
    with pytest.raises(TransportTimeout) as ex:
        a.run(10)
    t.join()
    # rank 1 marched iterations 1..4: its scalars reach rank 0's fold of
    # iteration 5, its halo of iteration 5 never comes
    entry = capi.build_plan(a.n, capi.neighbors(dims, 0), "v3")[0]
    stuck = 6 if fused else 5
    assert str(ex.value).startswith(f"rank 0: receive timed out at iteration {stuck}; outstanding: ")
    assert f"(src=1, tag={entry['recv_tag']})" in str(ex.value)
    a.close()
    b.close()


def test_seeded_rank_timing_is_deterministic():
    base = dict(grid=(24, 24, 24), steps=60, np=8, strategy="v3", overlap=1, check_every=10)
    plain = capi.run_case(capi.default_config(**base), collect_fields=True, collect_history=True)
    runs = [capi.run_case(capi.default_config(seed=s, **base), collect_fields=True, collect_history=True)
            for s in (20260131, 20260131, 7)]
    for r in runs:
        np.testing.assert_array_equal(bits(r.fields), bits(plain.fields))
        np.testing.assert_array_equal(bits(r.history), bits(plain.history))
        assert r.ledgers == plain.ledgers
    want = Oracle.run_case(capi.default_config(grid=(24, 24, 24), steps=60, check_every=10), collect_fields=True,
                           collect_history=True)
    np.testing.assert_array_equal(bits(plain.fields), bits(want["fields"]))


def _oracle_linf(n, steps, check_every, fluid, cfl=0.4):
    """max |R_v| over the interior at every check iteration of the oracle's
    serial loop (BC, residual, dt, update, rescale) from the quiescent state."""
    f = np.zeros((5, n[2] + 4, n[1] + 4, n[0] + 4))
    f[4] = fluid.t_inf
    h = capi.cavity_spacing(n)
    sp = O.stencil(h, fluid)
    box = ((2, 2, 2), (n[0] + 2, n[1] + 2, n[2] + 2))
    center = tuple((x - 1) // 2 + 2 for x in n)
    out = []
    for it in range(1, steps + 1):
        f = O.bc(f, n, (1,) * 6, fluid)
        r = O.residual(f, n, box, sp)
        if it == 1 or it % check_every == 0:
            inner = r[:, 2:n[2] + 2, 2:n[1] + 2, 2:n[0] + 2]
            out.append(np.abs(inner).reshape(5, -1).max(axis=1))
        dt = O.compute_dt(f, n, h, fluid, cfl)
        for v in range(5):
            f[v] = O.update(f[v], r[v], dt, n, box)
        f[0] = O.rescale(f[0], n, f[0][center[2], center[1], center[0]])
    return np.array(out)


@pytest.mark.parametrize("kw, env", [(dict(), {}), (dict(), {"CAV_STORED_GHOSTS": "1"}),
                                     (dict(np=2, mode="1d-i", strategy="v3", overlap=1), {}),
                                     (dict(np=4, mode="2d", strategy="v3", overlap=1), {"CAV_STORED_GHOSTS": "1"})])
def test_linf_norm_matches_numpy_over_oracle_residuals(monkeypatch, kw, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n = (24, 20, 16)
    cfg = capi.default_config(grid=n, steps=40, check_every=5, u_ref=1e-3, **kw)
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    want = _oracle_linf(n, 40, 5, cfg.fluid)
    assert r.history_linf.shape == want.shape
    np.testing.assert_array_equal(bits(r.history_linf), bits(want))
    assert np.all(want[1:] > 0)


def test_device_converged_solve_stored_ghosts(monkeypatch):
    monkeypatch.setenv("CAV_STORED_GHOSTS", "1")
    cfg = capi.default_config(grid=(32, 32, 32), steps=-1)  # configs[0]: converges at ~6600
    r = capi.run_case(cfg, collect_fields=True, collect_history=True)
    o = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    assert r.converged and o["converged"] and r.steps_marched == o["steps_marched"]
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    assert r.ledgers[0]["exchanges"] == r.steps_marched  # no ledger entries for the no-op tail


def test_gpu_scaling_series_csv(tmp_path):
    """run_bench on the GPU path (src/bench.cpp:18-75): strong and weak series
    in the reference's RunRecord CSV, validated, speedups filled against np=1,
    plus the B200 sidecar columns."""
    from paper_2006_02602_b200 import records, series
    for scaling in ("strong", "weak"):
        ser, extra, warn = series.run_series((24, 24, 24), [1, 2, 4], ["3d"], scaling=scaling, steps=6, warmup=2)
        assert not warn and len(ser) == 1 and [r.np for r in ser[0].rows] == [1, 2, 4]
        paths = series.write_outputs(ser, extra, str(tmp_path), scaling)
        rows = records.parse_csv(open(paths[0]).read())
        assert [r.np for r in rows] == [1, 2, 4]
        assert rows[0].speedup == 1.0 and rows[0].efficiency == 1.0
        assert all(r.ssspnt > 0 and r.steps == 6 for r in rows)
        if scaling == "weak":
            assert [r.size for r in rows] == [24 ** 3, 2 * 24 ** 3, 4 * 24 ** 3]
        side = open(paths[1]).read().splitlines()
        assert side[0] == series.EXTRA_HEADER and len(side) == 4
        assert extra[0]["roofline_frac"] > 0.0  # np = 1 owns its GPU
        assert all(0.0 < e["hbm_frac_of_step"] < 1.5 and e["exposed_comm_frac"] >= 0.0 for e in extra)


def test_ranks_on_one_hardware_queue():
    """Every stream of every in-process rank multiplexed onto ONE hardware
    queue (CUDA_DEVICE_MAX_CONNECTIONS=1, set before CUDA initialises in a
    fresh process): cross-rank waits are enqueued only after their
    producers, so even a single FIFO cannot deadlock; results stay bitwise."""
    import subprocess
    import sys
    import os
    code = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2006_02602_b200 import capi
from oracle.refbind import Oracle
for kw in (dict(np=4, mode="2d", strategy="v3", overlap=1), dict(np=3, mode="1d-j", strategy="v2", overlap=0),
           dict(np=8, mode="3d", strategy="baseline", overlap=1)):
    base = dict(grid=(26, 22, 18), steps=25, check_every=5)
    r = capi.run_case(capi.default_config(**base, **kw), collect_fields=True, collect_history=True)
    o = Oracle.run_case(capi.default_config(**base), collect_fields=True, collect_history=True)
    assert np.array_equal(r.fields.view(np.uint64), o["fields"].view(np.uint64)), kw
    assert np.array_equal(r.history.view(np.uint64), o["history"].view(np.uint64)), kw
print("ONE-QUEUE-OK")
""".format(root=os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0 and "ONE-QUEUE-OK" in p.stdout, p.stdout + p.stderr


_SOLVE_REF = {}


@pytest.mark.parametrize("kw", [dict(np=2, mode="1d-k", strategy="v3", overlap=1),
                                dict(np=4, mode="2d", strategy="v1", overlap=0),
                                dict(np=8, mode="3d", strategy="v3", overlap=1)])
def test_multi_rank_device_converged_solve(kw):
    """`cavity solve` on several ranks decided on the devices: after every
    check each rank pushes its exact norm digits to every rank, every rank
    merges them and applies the rule of src/runner.cpp:210-220 (no host round
    trip per check). Same converged iteration, history and fields as the
    oracle, and one exchange per marched iteration in every rank's ledger."""
    cfg = capi.default_config(grid=(32, 32, 32), steps=-1)
    if "o" not in _SOLVE_REF:
        _SOLVE_REF["o"] = Oracle.run_case(cfg, collect_fields=True, collect_history=True)
    o = _SOLVE_REF["o"]
    r = capi.run_case(capi.default_config(grid=(32, 32, 32), steps=-1, **kw), collect_fields=True,
                      collect_history=True)
    assert r.converged and o["converged"] and r.steps_marched == o["steps_marched"]
    assert list(r.history_iter) == list(o["history_iter"])
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]))
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]))
    assert all(l["exchanges"] == r.steps_marched for l in r.ledgers)


@pytest.mark.parametrize("dims, strategy, fused", [((2, 1, 1), "v3", "1"), ((1, 2, 2), "baseline", "1"),
                                                   ((2, 2, 2), "v3", "1"), ((2, 2, 2), "v1", "0")])
def test_multi_rank_blocks_from_uploaded_state(monkeypatch, dims, strategy, fused):
    """Several ranks start from an arbitrary uploaded state whose join ghosts
    are garbage: the exchange must replace them before the first residual
    (the reference exchanges every iteration before computing it), so the
    interiors after k steps equal the oracle's serial march of the global
    state. With fused halos this pins the prologue's initial-halo send
    (k_face_send) and the in-kernel halo stores from a developed state."""
    import threading
    monkeypatch.setenv("CAV_FUSED_HALO", fused)
    n = (24, 20, 18)
    gf = O.random_fields(n, 4242, vel=0.03)
    gf[0] *= 1e-3
    h = capi.cavity_spacing(n)
    np_ = dims[0] * dims[1] * dims[2]
    blocks = [capi.Block(r, np_, n, dims, strategy=strategy) for r in range(np_)]
    try:
        for b in blocks:
            for r in range(np_):
                if r != b.desc.rank:
                    b.connect(r, ptr=blocks[r].arena())
        for b in blocks:
            lo, m = b.lo, b.n
            local = gf[:, lo[2]:lo[2] + m[2] + 4, lo[1]:lo[1] + m[1] + 4, lo[0]:lo[0] + m[0] + 4].copy()
            for a, (l, hi_) in enumerate(((lo[0], lo[0] + m[0]), (lo[1], lo[1] + m[1]), (lo[2], lo[2] + m[2]))):
                sl = [slice(None)] * 4
                if l > 0:  # a joined low face: garbage in its ghost layers
                    sl[3 - a] = slice(0, 2)
                    local[tuple(sl)] = 7.0e3
                if hi_ < n[a]:
                    sl[3 - a] = slice(m[a] + 2, m[a] + 4)
                    local[tuple(sl)] = -7.0e3
            b.upload(local)
        errs = []

        def go(b, k):
            try:
                b.run(k)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        want = gf
        for k in (3, 4):
            ts = [threading.Thread(target=go, args=(b, k)) for b in blocks]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            assert not errs, errs
            want = O.march(want, n, h, capi.fluid_for_rayleigh(1e5), 0.4, k)
            for b in blocks:
                lo, m = b.lo, b.n
                got = b.download()[:, 2:m[2] + 2, 2:m[1] + 2, 2:m[0] + 2]
                exp = want[:, lo[2] + 2:lo[2] + m[2] + 2, lo[1] + 2:lo[1] + m[1] + 2, lo[0] + 2:lo[0] + m[0] + 2]
                np.testing.assert_array_equal(bits(got), bits(exp), err_msg=f"rank {b.desc.rank} after {k}")
    finally:
        for b in blocks:
            b.close()


def test_cpp_host_runs_the_case_through_the_c_abi(tmp_path):
    """The C++ host path north_star keeps: a g++-compiled driver includes
    include/cavity_b200.hpp, links libcavity_b200.so and runs cases (one rank,
    and two in-process ranks with fused halos); its fields and norm history
    equal the oracle's bitwise."""
    import shutil
    import subprocess
    import os
    if not shutil.which("g++"):
        pytest.skip("no g++")
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    src = tmp_path / "drv.cpp"
    src.write_text(r'''
#include <cstdio>
#include <cstdlib>
#include "cavity_b200.hpp"
int main(int argc, char** argv) {
  cav_run_config c = cavity_b200::default_config();
  c.nx = 24; c.ny = 20; c.nz = 16; c.steps = 60; c.check_every = 10;
  c.np = std::atoi(argv[1]); c.mode = CAV_MODE_1D_K;
  const cavity_b200::case_result r = cavity_b200::run_case(c, true, true);
  FILE* f = std::fopen(argv[2], "wb");
  std::fwrite(r.fields.data(), sizeof(double), r.fields.size(), f);
  std::fwrite(r.history.data(), sizeof(double), r.history.size(), f);
  std::fclose(f);
  std::printf("%lld %zu\n", r.raw.steps_marched, r.history_iter.size());
  return 0;
}''')
    exe = tmp_path / "drv"
    lib_dir = os.path.dirname(capi.lib_path())
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"), str(src), "-L", lib_dir,
                    "-lcavity_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    o = Oracle.run_case(capi.default_config(grid=(24, 20, 16), steps=60, check_every=10), collect_fields=True,
                        collect_history=True)
    for np_ in (1, 2):
        out = tmp_path / f"r{np_}.bin"
        p = subprocess.run([str(exe), str(np_), str(out)], capture_output=True, text=True, timeout=120,
                           env=dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32"))
        assert p.returncode == 0, p.stderr
        assert p.stdout.split() == ["60", str(len(o["history_iter"]))]
        data = np.fromfile(out, dtype=np.float64)
        nf = o["fields"].size
        np.testing.assert_array_equal(bits(data[:nf]), bits(o["fields"].ravel()))
        np.testing.assert_array_equal(bits(data[nf:]), bits(o["history"].ravel()))
