import json
import os
import subprocess
import sys

import pytest

# before anything initialises CUDA: several test ranks share one GPU
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


def _ensure_built():
    """Build the checkers and the sm_100a library if a previous build() did not."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libcavity_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if os.path.isdir("/root/reference/proj") and not os.path.exists(
            os.path.join(ROOT, "oracle", "_ref", "libcavity_ref.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2006_02602_b200", "lib", "libcavity_b200.so")):
        subprocess.run(["make", "-s", "-j4", "-C",
                        os.path.join(ROOT, "paper_2006_02602_b200", "csrc")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_arrays():
    import numpy as np
    return {
        "residual": dict(np.load(os.path.join(GOLDEN_DIR, "residual_random.npz"))),
        "runs": dict(np.load(os.path.join(GOLDEN_DIR, "runs_small_fields.npz"))),
    }


def golden_config(entry, default_config):
    """Rebuild a RunConfig from a golden run entry."""
    kw = dict(entry["config"])
    if "grid" in kw:
        kw["grid"] = tuple(kw["grid"])
    cfg = default_config(**kw)
    if "sigma" in entry:
        cfg.fluid.sigma = float.fromhex(entry["sigma"])
    return cfg
