"""Seeded stress corpora shared by the golden generator (tests/golden/make_stress_golden.py,
which runs the REAL reference on them) and the GPU parity tests.  Pure numpy plus the
oracle's C generator (test infrastructure); nothing here reads /root/reference."""

import ctypes

import numpy as np


def edge_corpus(n, eb, seed, x0=0.37, n_bins_half=32768):
    """SURVEY.md 8.P adversarial corpus: every x_i within 0..3 ulps of a bin edge of the
    reference chain's own prediction (about half the open-loop codes disagree)."""
    from oracle import oracle as orc
    r = np.random.default_rng(seed)
    m = r.integers(-40, 41, size=n - 1).astype(np.int64)
    k = r.integers(-3, 4, size=n - 1).astype(np.int64)
    out = np.empty(n, dtype=np.float64)
    L = orc.lib()
    f = L.lco_edge_corpus
    f.restype = None
    f.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                  ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
    f(m.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), k.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
      n, x0, eb, n_bins_half, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def int_walk(n, seed, step=5):
    """Integer-valued random walk (exactly representable chain at eb = 0.5: every
    prediction error is an integer, q = m + 0.5 lands exactly on a bin midpoint)."""
    r = np.random.default_rng(seed)
    return np.cumsum(r.integers(-step, step + 1, size=n)).astype(np.float64)


def fib_walk(n_sym, seed):
    """Integer walk whose increments take n_sym distinct values with Fibonacci
    frequencies F_1..F_n_sym (shuffled): at eb = 0.5 the codes follow that
    distribution exactly, so the Huffman tree has depth n_sym - 1 (n_sym = 35:
    24,157,816 symbols, codes up to 34 bits -- the encoder's and decoder's
    >32-bit paths)."""
    fib = [1, 1]
    while len(fib) < n_sym:
        fib.append(fib[-1] + fib[-2])
    # increments 0, -1, 1, -2, 2, ... (codes 1, 2, 3, ...): zigzag order
    incs = np.array([(j + 1) // 2 * (1 if j % 2 == 0 else -1) if j else 0 for j in range(n_sym)], np.int64)
    steps = np.repeat(incs, fib)
    np.random.default_rng(seed).shuffle(steps)
    x = np.concatenate([[0], np.cumsum(steps)]).astype(np.float64)
    return x


def sine_mix(n, seed):
    """Config-2 generator (BASELINE.json configs[1]) at any n."""
    r = np.random.default_rng(seed)
    f = r.uniform(1, 64, 8)
    a = r.uniform(0, 1, 8)
    ph = r.uniform(0, 2 * np.pi, 8)
    t = np.arange(n) / n
    x = np.zeros(n)
    for k in range(8):
        x += a[k] * np.sin(2 * np.pi * f[k] * t + ph[k])
    return x + r.normal(0, 1e-3, n)


# (name, generator, mode, eb, n_bins_half) -- the stress cases the golden file pins
CASES = [
    ("edge2m_a", lambda: edge_corpus(1 << 21, 1e-3, 201), "absolute", 1e-3, 32768),
    ("edge4m_b", lambda: edge_corpus(1 << 22, 3.7e-5, 202, x0=-1.25), "absolute", 3.7e-5, 32768),
    ("edge1m_c", lambda: edge_corpus(1 << 20, 1e-7, 203, x0=1e3), "absolute", 1e-7, 32768),
    ("edge1m_nb32", lambda: edge_corpus(1 << 20, 2e-4, 204, n_bins_half=32), "absolute", 2e-4, 32),
    ("intwalk4m_half", lambda: int_walk(1 << 22, 205), "absolute", 0.5, 32768),
    ("intwalk2m_rel", lambda: int_walk(1 << 21, 206, step=40), "value_range_relative", 1e-4, 32768),
    ("fib35", lambda: fib_walk(35, 207), "absolute", 0.5, 32768),
]
