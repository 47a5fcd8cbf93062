"""Host-side check of the chunked exact-chain algorithm (test infrastructure).

Builds tests/cpu/chain_sim.cpp (which includes the product header
paper_1805_07384_b200/csrc/lc_chain.cuh compiled for the host) and checks, on
seeded vectors, that (1) the deferred event tracker + replay reproduces the
step-by-step offset map of every chunk and (2) the predicted chunk starts
match the sequential reference chain (compressor.py:358-376 recurrence).
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "chain_sim.so")

f64p = ctypes.POINTER(ctypes.c_double)
i64p = ctypes.POINTER(ctypes.c_int64)


def build():
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    src = os.path.join(HERE, "chain_sim.cpp")
    if not os.path.exists(SO) or os.path.getmtime(SO) < max(
            os.path.getmtime(src),
            os.path.getmtime(os.path.join(HERE, "..", "..", "paper_1805_07384_b200", "csrc", "lc_chain.cuh"))):
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-shared", "-fPIC", "-o", SO, src])
    L = ctypes.CDLL(SO)
    L.sim_predict.restype = ctypes.c_int64
    L.sim_predict.argtypes = [f64p, ctypes.c_int64, ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                              i64p, i64p]
    return L


def predict(L, x, eb, nbh=32768, mode=0, chunk=32):
    """-> (bad chunks, first bad, true map changes, flagged steps, chunks); flagged < 0: tracker mismatch."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    fb, ne = ctypes.c_int64(), ctypes.c_int64()
    bad = L.sim_predict(x.ctypes.data_as(f64p), x.size, eb, nbh, chunk, mode, ctypes.byref(fb), ctypes.byref(ne))
    ev = ne.value
    if ev < 0:
        return bad, fb.value, -1, -1, (x.size - 1 + chunk - 1) // chunk
    return bad, fb.value, ev // 1000000, ev % 1000000, (x.size - 1 + chunk - 1) // chunk


def vectors(seed=0, n=1 << 16):
    r = np.random.default_rng(seed)
    t = np.arange(n) / n
    out = {}
    s = np.zeros(n)
    for _ in range(8):
        s += r.uniform(0, 1) * np.sin(2 * np.pi * r.uniform(1, 64) * t + r.uniform(0, 2 * np.pi))
    out["sine"] = (s + r.normal(0, 1e-3, n), [1e-3, 1e-4, 1e-6])
    # dyadic steps around 2^30: rounding ties of r + m*delta are frequent
    d = 3.0 * 2.0 ** -30
    w = 2.0 ** 30 + np.cumsum(r.integers(-300, 300, n)) * d + r.normal(0, 1e-6, n)
    out["tie_2p30"] = (w, [1.5 * 2.0 ** -30 / (w.max() - w.min())])
    # crossing powers of two and zero, integer-valued data
    out["cross"] = (np.cumsum(r.normal(0, 0.05, n)) + 1.0, [1e-3, 1e-6])
    out["ints"] = (np.round(np.cumsum(r.normal(0, 3, n))), [0.5 / 1000, 1e-6])
    out["zeros"] = (np.concatenate([np.zeros(n // 2), r.normal(0, 1, n - n // 2)]), [1e-4])
    return out


if __name__ == "__main__":
    L = build()
    for name, (x, ebs) in vectors().items():
        vr = float(x.max() - x.min())
        for ebr in ebs:
            for mode in (0, 1):
                print(name, ebr, mode, predict(L, x, ebr * vr, mode=mode))
