import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


def golden_block_names(z):
    return sorted({k.split("/")[0] for k in z.files
                   if k.endswith("/block")})


MODES = {0: "absolute", 1: "value_range_relative", 2: "fixed_psnr"}


REF_PATH = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="session")
def reference():
    """The real reference package (lossyckpt) installed under baseline/_ref
    (python -m pip install --no-deps --target baseline/_ref <copy of the
    reference>; gitignored, travels with the repo snapshot).  Skips when absent."""
    if os.path.isdir(os.path.join(REF_PATH, "lossyckpt")) and REF_PATH not in sys.path:
        sys.path.append(REF_PATH)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "lc_numba_cache"))
    return pytest.importorskip("lossyckpt")
