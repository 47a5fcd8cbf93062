"""Generate CKPTIMG1 golden images with the REAL reference checkpoint layer.

Run in the build container (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_ckpt_golden.py

Writes tests/golden/ckpt_golden.npz: for each case the input vector, the
iteration, the compressor mode/parameter (lossy cases) and the bytes of the
image the reference writes through StorageTarget(path=...).commit
(checkpoint.py:110-119, 150-177).
"""

import os
import sys
import tempfile
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lossyckpt import checkpoint as ck  # noqa: E402
from lossyckpt import compressor as cp  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ckpt_golden.npz")
rng = np.random.default_rng(2024)
cases = {}


def image_bytes(image):
    with tempfile.TemporaryDirectory() as d:
        target = ck.StorageTarget(path=os.path.join(d, "img"))
        target.commit(image)
        return open(os.path.join(d, "img"), "rb").read()


def add_raw(name, x, it):
    img, _ = ck.checkpoint_traditional(SimpleNamespace(x=x, iteration=it), ck.StorageTarget(), commit=False)
    cases[name + "/x"] = x
    cases[name + "/meta"] = np.array([it, 0, 0, 0], dtype=np.float64)
    cases[name + "/image"] = np.frombuffer(image_bytes(img), dtype=np.uint8)


def add_lossy(name, x, it, mode, param):
    cfg = {0: cp.CompressorConfig.absolute, 1: cp.CompressorConfig.value_range_relative,
           2: cp.CompressorConfig.fixed_psnr}[mode](param)
    img, _ = ck.checkpoint_lossy(SimpleNamespace(x=x, iteration=it), cfg, ck.StorageTarget(), commit=False)
    cases[name + "/x"] = x
    cases[name + "/meta"] = np.array([it, 1, mode, param], dtype=np.float64)
    cases[name + "/image"] = np.frombuffer(image_bytes(img), dtype=np.uint8)
    cases[name + "/recon"] = ck.decode_payload(img)


t = np.arange(1 << 14) / (1 << 14)
smooth = np.sin(2 * np.pi * 3 * t) + 0.25 * np.cos(2 * np.pi * 17 * t) + rng.normal(0, 1e-3, t.size)
add_raw("raw_small", rng.normal(size=257), 7)
add_raw("raw_one", np.array([3.25]), 0)
add_lossy("lossy_rel4", smooth, 42, 1, 1e-4)
add_lossy("lossy_abs", smooth * 1e3, 190, 0, 1e-2)
add_lossy("lossy_psnr", smooth, 5, 2, 80.0)
add_lossy("lossy_const", np.full(100, 1.5), 11, 1, 1e-3)
walk = np.cumsum(rng.normal(0, 1, 5000))
walk[::997] += 1e6                                    # escapes
add_lossy("lossy_esc", walk, 3, 1, 1e-6)
np.savez_compressed(OUT, **cases)
print("wrote", OUT, len(cases), "arrays")
