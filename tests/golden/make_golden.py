"""Generate golden vectors by running the REAL reference (lossyckpt, Python+numba).

Run in the build container (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Each case stores the input vector (each
distinct vector once, under vec/<k>), the compressor config, the reference's
serialized block (CompressedBlock.to_bytes) and the sha256 of its
reconstruction (compressor.decompress).  Inputs are stored (not just seeds) so
parity never depends on numpy's distribution algorithms.

Corpora:
  ident_*   the criterion-5 identity corpus (test_acceptance.py:91-105, seed 55)
  crit6_*   the first pairs of the criterion-6 corpus (test_acceptance.py:108-134)
  edge_*    an adversarial bin-edge corpus: x_i placed at r_{i-1}+(m-1/2)*delta +- k ulp
  jac190_*  config 1's checkpoint vector: Jacobi on poisson2d(256), b~U(-1,1) seed 0,
            x at iteration 190 (BASELINE.json configs[0])
  sine_*    config 2's generator at n=2^16
  huff_*    Huffman code_lengths on adversarial frequency tables + decode error statuses
"""

import hashlib
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lossyckpt import compressor as cp  # noqa: E402
from lossyckpt import fields, huffman, solvers, sparse  # noqa: E402
from lossyckpt.errors import IntegrityError  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
cases = {}
_vec_ids = {}


def _vec(data):
    """Store each distinct input vector once; return its key."""
    key = hashlib.sha256(data.tobytes()).hexdigest()[:16]
    if key not in _vec_ids:
        _vec_ids[key] = f"vec/{len(_vec_ids)}"
        cases[_vec_ids[key]] = data
    return _vec_ids[key]


def add_block(name, data, mode, param, n_bins_half=32768):
    data = np.ascontiguousarray(data, dtype=np.float64)
    if mode == "absolute":
        cfg = cp.CompressorConfig.absolute(param, n_bins_half=n_bins_half)
    elif mode == "value_range_relative":
        cfg = cp.CompressorConfig.value_range_relative(param, n_bins_half=n_bins_half)
    else:
        cfg = cp.CompressorConfig.fixed_psnr(param, n_bins_half=n_bins_half)
    block = cp.compress(data, cfg)
    blob = block.to_bytes()
    recon = cp.decompress(block)
    cases[f"{name}/x"] = np.array(_vec(data))
    cases[f"{name}/cfg"] = np.array([{"absolute": 0, "value_range_relative": 1, "fixed_psnr": 2}[mode],
                                     param, n_bins_half], dtype=np.float64)
    cases[f"{name}/block"] = np.frombuffer(blob, dtype=np.uint8)
    cases[f"{name}/recon_sha256"] = np.array(hashlib.sha256(recon.tobytes()).hexdigest())


# --- criterion-5 identity corpus --------------------------------------------
rng = np.random.default_rng(55)
corpus = [d for _, d in fields.smooth_field_corpus(n=2048, seed=3)]
corpus.append(rng.normal(size=10_000).cumsum())
corpus.append(rng.normal(size=4096) * 1e6)
corpus.append(np.full(512, math.pi))
spiky = rng.normal(size=2048).cumsum()
spiky[::100] += 1e9
corpus.append(spiky)
for i, d in enumerate(corpus):
    add_block(f"ident_{i}_r3", d, "value_range_relative", 1e-3)
    add_block(f"ident_{i}_r6", d, "value_range_relative", 1e-6)
    add_block(f"ident_{i}_p80", d, "fixed_psnr", 80.0)

# --- criterion-6 corpus (first 100 pairs) -------------------------------------
rng = np.random.default_rng(66)
for p in range(100):
    kind = p % 4
    size = int(rng.integers(2, 1500))
    if kind == 0:
        data = fields.sine_mixture(max(size, 8), n_modes=3, seed=int(rng.integers(1e9)))
    elif kind == 1:
        data = rng.normal(size=size).cumsum()
    elif kind == 2:
        data = rng.normal(size=size) * 10.0 ** rng.integers(-3, 9)
    else:
        data = rng.normal(size=size).cumsum()
        data[rng.integers(0, size)] += 10.0 ** rng.integers(3, 12)
    eb = 10.0 ** rng.uniform(-9, 2)
    add_block(f"crit6_{p}", data, "absolute", float(eb))


# --- adversarial bin-edge corpus ---------------------------------------------
def edge_corpus(n, eb, seed, x0=0.37):
    """Advance a reference-exact chain and put each x_i within a few ulps of a bin edge."""
    r = np.random.default_rng(seed)
    delta = 2.0 * eb
    xs = [x0]
    prev = x0
    for _ in range(n - 1):
        m = int(r.integers(-40, 41))
        edge = prev + (m - 0.5) * delta
        k = int(r.integers(-3, 4))
        v = float(edge)
        for _ in range(abs(k)):
            v = math.nextafter(v, math.inf if k > 0 else -math.inf)
        xs.append(v)
        # advance with the reference semantics (compressor.py:329-351)
        pe = v - prev
        q = pe / delta + 0.5
        esc = True
        cand = prev
        if -32767.0 <= q < 32768.0:
            mm = math.floor(q)
            cand = prev if mm == 0 else prev + mm * delta
            if abs(v - cand) <= eb:
                esc = False
        prev = v if esc else cand
    return np.array(xs)


for s, eb in enumerate((1e-3, 3.7e-5, 1e-7)):
    add_block(f"edge_{s}", edge_corpus(6000, eb, 100 + s), "absolute", eb)

# --- config 1 checkpoint vector (Jacobi, poisson2d(256), iteration 190) ------
a, _ = sparse.generate_poisson2d(256)
prec = sparse.jacobi_preconditioner(a)
b = np.random.default_rng(0).uniform(-1.0, 1.0, 256 * 256)
st = solvers.init("jacobi", a, prec, b, solvers.SolveConfig(tolerance=1e-6, max_iterations=200_000,
                                                          restart_len=10, ckpt_intvl=10))
while st.iteration < 190:
    st.step()
x190 = st.x.copy()
for tag, eb in (("r4", 1e-4), ("r5", 1e-5), ("r6", 1e-6)):
    add_block(f"jac190_{tag}", x190, "value_range_relative", eb)

# --- config 2 generator at n = 2^16 -----------------------------------------
n = 1 << 16
r = np.random.default_rng(0)
f = r.uniform(1, 64, 8)
amp = r.uniform(0, 1, 8)
ph = r.uniform(0, 2 * np.pi, 8)
t = np.arange(n) / n
x = (amp[None, :] * np.sin(2 * np.pi * f[None, :] * t[:, None] + ph[None, :])).sum(1) + r.normal(0, 1e-3, n)
for tag, eb in (("r3", 1e-3), ("r4", 1e-4), ("r6", 1e-6)):
    add_block(f"sine_{tag}", x, "value_range_relative", eb)

# small-bin-budget and tiny cases
add_block("nb1_walk", np.random.default_rng(5).normal(size=300).cumsum(), "absolute", 0.5, n_bins_half=1)
add_block("nb7_walk", np.random.default_rng(6).normal(size=300).cumsum(), "absolute", 0.05, n_bins_half=7)
add_block("two_elems", np.array([1.0, 2.0]), "absolute", 0.1)
add_block("single", np.array([42.0]), "absolute", 1.0)
add_block("negzero", np.array([-0.0, -0.0, 1e-300, -0.0, 0.0, 5e-324]), "absolute", 1e-3)

# --- Huffman code_lengths on adversarial tables -------------------------------
r = np.random.default_rng(7)
tables = []
tables.append(np.array([1, 1, 2]))
tables.append(np.array([5, 5, 5, 5]))
fib = [1, 1]
while len(fib) < 40:
    fib.append(fib[-1] + fib[-2])
tables.append(np.array(fib))                        # Fibonacci -> deep tree
tables.append(np.array(fib[::-1]))
for _ in range(60):
    k = int(r.integers(2, 300))
    t_ = r.integers(0, 6, size=k) * (r.random(k) < 0.7)   # heavy ties and zeros
    tables.append(t_)
for _ in range(20):
    k = int(r.integers(2, 2000))
    tables.append(np.floor(r.pareto(1.2, size=k) * 10).astype(np.int64))
for i, tb in enumerate(tables):
    cases[f"huff_{i}/freqs"] = np.asarray(tb, dtype=np.int64)
    cases[f"huff_{i}/lengths"] = huffman.code_lengths(np.asarray(tb, dtype=np.int64))

# --- decode error statuses ----------------------------------------------------
r = np.random.default_rng(8)
errs = []
for i in range(40):
    syms = r.integers(0, 16, size=int(r.integers(5, 400)))
    lengths = huffman.code_lengths(np.bincount(syms, minlength=16))
    payload, bits = huffman.encode(syms, lengths)
    kind = i % 4
    count = len(syms)
    if kind == 0:           # truncate bit length
        bits2 = max(1, bits - int(r.integers(1, 9)))
        payload2 = payload[: (bits2 + 7) // 8]
    elif kind == 1:         # extra trailing bits
        bits2 = bits + int(r.integers(1, 9))
        payload2 = payload + b"\x00"
    elif kind == 2:         # fewer symbols requested than encoded -> trailing bits
        bits2, payload2 = bits, payload
        count = count - int(r.integers(1, 4))
    else:                   # wrong codebook (incomplete code)
        bits2, payload2 = bits, payload
        lengths = huffman.code_lengths(np.arange(1, 5))
    try:
        out = huffman.decode(payload2, bits2, lengths, count)
        status = "ok"
    except IntegrityError as e:
        status = str(e)
        out = np.zeros(0, np.int64)
    cases[f"derr_{i}/payload"] = np.frombuffer(payload2, dtype=np.uint8)
    cases[f"derr_{i}/bits"] = np.array([bits2, count], dtype=np.int64)
    cases[f"derr_{i}/lengths"] = lengths
    cases[f"derr_{i}/status"] = np.array(status)
    cases[f"derr_{i}/out"] = out

np.savez_compressed(OUT, **cases)
print(f"wrote {OUT}: {len(cases)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")
