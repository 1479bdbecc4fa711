"""BASELINE.json's configs at their real sizes and lengths, bitwise.

* C1 (configs[1]): 256^3 x 2000 iterations with the 201-sample residual-norm
  history, against the unmodified reference's own run_case (oracle/_ref) on
  the host cores. The reference is bitwise decomposition-independent
  (P/README.md:10-15), so its threads-as-ranks run IS the serial answer
  (acceptance c1 model, tests/acceptance.cpp:144-153).
* 512^3 on one GPU pinned to the reference for 10 iterations (norms at every
  step), which makes the GPU np=1 run the comparison point for the
  decompositions below.
* C2 (configs[2]): 256^3, 1d-i slabs at np = 2, 4, 8 (non-contiguous faces),
  V3, overlap on.
* C3 (configs[3]): 512^3, 2d (1,2,2) / (1,2,4) and 3d (2,2,2), V3, overlap on.
* C4 (configs[4]): grow_grid(256^3, np, 3d, type 2) (src/decomp.cpp:227-255):
  256^2x512 (np 2), 256x512^2 (np 4), 512^3 (np 8).

Decomposed runs put every rank on device 0 (the in-process block group is the
multi-GPU code path: peer pointers, remote ghost stores, stream-ordered
waits). They march 20-50 iterations with history and must reproduce the GPU
np=1 run of the same grid bit for bit (fields and norms).
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.refbind import Ref, ref_available
from paper_2006_02602_b200 import _abi, capi

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def ref_np(grid, mode="3d"):
    """Largest np <= host cores that the reference's own choose_dims/partition
    accept for `grid` (threads-as-ranks, its only parallelism)."""
    L = Ref.lib()
    np_ = min(os.cpu_count() or 1, 64)
    while np_ > 1:
        dims = (C.c_int * 3)()
        if L.ref_choose_dims(np_, _abi.MODES[mode], dims) == 0:
            ext = (C.c_int * (6 * np_))()
            if L.ref_partition(grid[0], grid[1], grid[2], dims, ext) == 0:
                return np_
        np_ -= 1
    return 1


def run_ref(grid, steps, check_every):
    np_ = ref_np(grid)
    cfg = capi.default_config(grid=grid, steps=steps, check_every=check_every, np=np_, mode="3d")
    return Ref.run_case(cfg, collect_fields=True, collect_history=True)


def run_gpu(grid, steps, check_every, **kw):
    cfg = capi.default_config(grid=grid, steps=steps, check_every=check_every, **kw)
    return capi.run_case(cfg, collect_fields=True, collect_history=True)


def assert_same(got, want, what):
    assert list(got.history_iter) == list(want["history_iter"]), what
    np.testing.assert_array_equal(bits(got.history), bits(want["history"]), err_msg=what)
    np.testing.assert_array_equal(bits(got.fields), bits(want["fields"]), err_msg=what)


@needs_ref
def test_c1_256cube_2000_iterations_matches_reference():
    """configs[1] exactly: 256^3, 2000 iterations, norm history every 10th
    (201 samples) — fields and history bitwise equal to the reference."""
    want = run_ref((256, 256, 256), 2000, 10)
    got = run_gpu((256, 256, 256), 2000, 10)
    assert len(got.history_iter) == 201 and got.steps_marched == 2000
    assert_same(got, want, "C1 256^3 x 2000")
    # the decomposition-independent reference fields, also as the GPU's
    # linf/l2 sanity: the flow developed (not the quiescent state)
    assert np.abs(got.fields[1]).max() > 1e-4


_cache = {}


def gpu_serial(grid, steps, check_every):
    key = (grid, steps, check_every)
    if key not in _cache:
        _cache.clear()  # one grid at a time (512^3 fields are 5.4 GB)
        _cache[key] = run_gpu(grid, steps, check_every)
    return _cache[key]


@needs_ref
def test_512cube_single_gpu_pinned_to_reference():
    """The np=1 512^3 run that the C3/C4 decompositions are compared with is
    itself bitwise equal to the reference (10 iterations, norms every step)."""
    want = run_ref((512, 512, 512), 10, 1)
    got = run_gpu((512, 512, 512), 10, 1)
    assert_same(got, want, "512^3 x 10")


@pytest.mark.parametrize("np_", [2, 4, 8])
def test_c2_256cube_1d_i_slabs(np_):
    """configs[2]: 1d-i slabs (i-faces are the non-contiguous ones), V3
    per-variable halo depth, overlap on; 50 iterations, history every 5."""
    want = gpu_serial((256, 256, 256), 50, 5)
    got = run_gpu((256, 256, 256), 50, 5, np=np_, mode="1d-i", strategy="v3", overlap=1)
    assert got.dims == (np_, 1, 1)
    assert_same(got, {"history_iter": want.history_iter, "history": want.history, "fields": want.fields},
                f"C2 1d-i np={np_}")


@pytest.mark.parametrize("np_, mode, dims", [(4, "2d", (1, 2, 2)), (8, "2d", (1, 2, 4)), (8, "3d", (2, 2, 2))])
def test_c3_512cube_2d_3d(np_, mode, dims):
    """configs[3]: 512^3 with 2d and 3d block decompositions, V3, overlap on;
    20 iterations, history every 5."""
    want = gpu_serial((512, 512, 512), 20, 5)
    got = run_gpu((512, 512, 512), 20, 5, np=np_, mode=mode, strategy="v3", overlap=1)
    assert got.dims == dims
    assert_same(got, {"history_iter": want.history_iter, "history": want.history, "fields": want.fields},
                f"C3 {mode} np={np_}")


@pytest.mark.parametrize("np_, grid", [(2, (256, 256, 512)), (4, (256, 512, 512)), (8, (512, 512, 512))])
def test_c4_weak_grow_grid(np_, grid):
    """configs[4]: weak scaling at 256^3 per GPU, 3d decomposition, grids from
    the reference's grow_grid type 2; per-variable halo depth (V3)."""
    assert capi.grow_grid((256, 256, 256), np_, "3d", 2) == grid
    want = gpu_serial(grid, 20, 5)
    got = run_gpu(grid, 20, 5, np=np_, mode="3d", strategy="v3", overlap=1)
    assert got.dims[0] * got.dims[1] * got.dims[2] == np_
    assert_same(got, {"history_iter": want.history_iter, "history": want.history, "fields": want.fields},
                f"C4 {grid} np={np_}")
