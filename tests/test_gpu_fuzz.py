"""Seeded random configurations through the whole GPU path vs the oracle,
bitwise (the reference is decomposition-, strategy- and overlap-independent
bit for bit, P/README.md:10-15, so the serial oracle is the expected result
for every draw). Covers odd and ragged grids (tile edges, partial tiles,
odd box origins), every decomposition mode and strategy, overlap on/off,
the adaptive k-chunk and tail chunks, small and large rank counts, and
several check cadences."""
import random

import numpy as np
import pytest

from oracle.refbind import Oracle
from paper_2006_02602_b200 import capi

pytestmark = pytest.mark.gpu

MODES = ["1d-i", "1d-j", "1d-k", "2d", "3d"]
STRATEGIES = ["baseline", "v1", "v2", "v3"]


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def draw(seed):
    rng = random.Random(seed)
    grid = tuple(rng.randint(5, 72) for _ in range(3))
    for _ in range(50):
        np_ = rng.choice([1, 1, 2, 3, 4, 6, 8])
        mode = rng.choice(MODES)
        try:
            dims = capi.choose_dims(np_, mode)
            capi.partition(grid, dims)
            break
        except Exception:
            continue
    else:
        np_, mode = 1, "3d"
    return dict(grid=grid, steps=rng.randint(6, 24), check_every=rng.choice([1, 3, 5, 10]), np=np_, mode=mode,
                strategy=rng.choice(STRATEGIES), overlap=rng.randint(0, 1), u_ref=rng.choice([0.03, 0.03, 1e-3]))


@pytest.mark.parametrize("seed", list(range(48)))
@pytest.mark.parametrize("ghosts", ["auto", "1", "slab"])
def test_random_configuration_matches_oracle(monkeypatch, seed, ghosts):
    """ghosts "1" forces the stored-wall-ghost step on every draw (by default
    it starts at 3e6 cells per block, above these grids); "slab" runs the
    multi-rank draws through the pack/unpack slab exchange instead of the
    step kernel's fused halo stores."""
    monkeypatch.setenv("CAV_STORED_GHOSTS", "1" if ghosts == "1" else "-1")
    monkeypatch.setenv("CAV_FUSED_HALO", "0" if ghosts == "slab" else "1")
    kw = draw(seed)
    r = capi.run_case(capi.default_config(**kw), collect_fields=True, collect_history=True)
    serial = {k: v for k, v in kw.items() if k not in ("np", "mode", "strategy", "overlap")}
    o = Oracle.run_case(capi.default_config(**serial), collect_fields=True, collect_history=True)
    assert list(r.history_iter) == list(o["history_iter"]), kw
    np.testing.assert_array_equal(bits(r.history), bits(o["history"]), err_msg=str(kw))
    np.testing.assert_array_equal(bits(r.fields), bits(o["fields"]), err_msg=str(kw))
