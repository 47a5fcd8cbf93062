"""Exactness under stress, on the GPU (VERDICT r1 "next round" item 1).

* Large adversarial corpora (every x_i within 0..3 ulps of a bin edge of the reference
  chain; integer walks at eb = 0.5; a Fibonacci-distributed stream whose
  Huffman codes reach 34 bits) against sha256 hashes of the REAL reference's blocks and
  reconstructions (tests/golden/make_stress_golden.py, tests/golden/stress_golden.json).
* Every fallback path forced and checked bit-exact: quantizer relaunch, quantizer
  sequential chain, decoder relaunch, decoder sequential chain.
* The 84 adversarial Huffman tables of the golden file through the device codebook.
"""

import ctypes
import hashlib
import json
import os
import sys

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import stress_inputs  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "stress_golden.json")))

OPT_MAX_QUANT, OPT_MAX_REC, OPT_INJECT_QUANT, OPT_INJECT_REC, OPT_VERIFY, OPT_RESUME = 0, 1, 2, 3, 4, 5
STAT_QUANT_RELAUNCHES, STAT_QUANT_SERIAL, STAT_REC_RELAUNCHES, STAT_REC_SERIAL = 0, 1, 2, 3


@pytest.fixture(scope="module")
def lc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_07384_b200 as lc
    return lc


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def _cfg(lc, mode, eb, nbh):
    if mode == "absolute":
        return lc.CompressorConfig.absolute(eb, n_bins_half=nbh)
    return lc.CompressorConfig.value_range_relative(eb, n_bins_half=nbh)


@pytest.fixture
def ctx(lc):
    from paper_1805_07384_b200 import _native
    c = _native.context(0)
    yield c
    for k, v in ((OPT_MAX_QUANT, 64), (OPT_MAX_REC, 64), (OPT_INJECT_QUANT, -1), (OPT_INJECT_REC, -1),
                 (OPT_VERIFY, 0), (OPT_RESUME, 1)):
        c.lib.lc_ctx_set_option(c.h, k, v)


@pytest.mark.parametrize("case", [c[0] for c in stress_inputs.CASES])
@pytest.mark.parametrize("verify", [0, 1])
def test_stress_corpus_matches_reference(lc, ctx, case, verify):
    """Block bytes and reconstruction identical to the real reference's (sha256), with
    the quantizer's certified fast path (verify=0) and with every chunk re-run by the
    exact reference step and end-checked (verify=1)."""
    name, gen, mode, eb, nbh = next(c for c in stress_inputs.CASES if c[0] == case)
    g = GOLD[name]
    x = gen()
    assert _sha(x.tobytes()) == g["x_sha256"], "input generator drifted"
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_VERIFY, verify)
    blk = lc.compress(torch.from_numpy(x).cuda(), _cfg(lc, mode, eb, nbh))
    data = blk.to_bytes()
    assert len(blk.escape_indices) == g["n_esc"]
    assert int(np.asarray(blk.code_lengths).max()) == g["max_len"]
    assert _sha(data) == g["block_sha256"], (name, ctx.lib.lc_ctx_get_stat(ctx.h, STAT_QUANT_RELAUNCHES))
    rec = lc.decompress(lc.CompressedBlock.from_bytes(data))
    assert _sha(rec.tobytes()) == g["recon_sha256"], name
    assert np.all(np.abs(rec - x) <= blk.eb_abs)


def _edge(n=300_000):
    return stress_inputs.edge_corpus(n, 1e-3, 301)


def _smooth(n=300_000):
    return stress_inputs.sine_mix(n, 302)


@pytest.mark.parametrize("max_relaunch,resume", [(64, 1), (64, 0), (0, 1)])
def test_quantizer_relaunch_and_serial_paths(lc, ctx, max_relaunch, resume):
    """A wrong chunk prediction (injected) is caught by its predecessor's end check and
    repaired by resuming the exact pass from the failing chunk (resume 1, the default),
    a full relaunch (resume 0) or the sequential exact chain (max 0); the block is the
    oracle's every way.  (Smooth data: the injected failure is the only one.)"""
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_RESUME, resume)
    x = _smooth()
    ref = orc.to_bytes(orc.compress(x, "absolute", 1e-3))
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_INJECT_QUANT, -1)
    lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.absolute(1e-3))
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_QUANT_RELAUNCHES) == 0      # no failure without injection
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_VERIFY, 1)           # every chunk end-checked
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_INJECT_QUANT, 5000)
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_MAX_QUANT, max_relaunch)
    blk = lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.absolute(1e-3))
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_QUANT_RELAUNCHES) == 1
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_QUANT_SERIAL) == (1 if max_relaunch == 0 else 0)
    assert blk.to_bytes() == ref


@pytest.mark.parametrize("max_relaunch", [64, 0])
def test_decoder_relaunch_and_serial_paths(lc, ctx, max_relaunch):
    """The same for the decoder's reconstruction (compressor.py:358-376): the injected
    misprediction is repaired by a relaunch or the sequential chain, x' is bit-identical,
    and the escape checks (count, positions) still run on the serial path."""
    x = _smooth()
    x[[1000, 77_777, 250_001]] += 1e6                         # escapes
    d = orc.compress(x, "absolute", 1e-3)
    blk = lc.CompressedBlock.from_bytes(orc.to_bytes(d))
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_INJECT_REC, 4321)
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_MAX_REC, max_relaunch)
    rec = lc.decompress(blk)
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_REC_RELAUNCHES) == 1
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_REC_SERIAL) == (1 if max_relaunch == 0 else 0)
    assert np.array_equal(rec.view(np.int64), d["recon"].view(np.int64))
    import dataclasses
    moved = dataclasses.replace(blk, escape_indices=blk.escape_indices + 1)
    with pytest.raises(lc.IntegrityError, match="escape positions disagree"):
        lc.decompress(moved)


def test_golden_huffman_tables_on_device(lc, ctx, golden):
    """huffman.code_lengths + canonical_codes (huffman.py:21-72) on the device codebook for
    the 84 adversarial reference tables: heavy ties, zeros, Fibonacci depths up to 39."""
    names = sorted(k[:-6] for k in golden.files if k.startswith("huff_") and k.endswith("/freqs"))
    assert len(names) == 84
    deepest = 0
    for nm in names:
        f = golden[nm + "/freqs"].astype(np.int64)
        want = golden[nm + "/lengths"].astype(np.uint8)
        nb = max(2, 1 << int(np.ceil(np.log2(max(f.size, 2)))))
        hist = np.zeros(nb, np.uint32)
        hist[:f.size] = f
        lengths = np.zeros(nb, np.uint8)
        codes = np.zeros(nb, np.uint64)
        ml = ctypes.c_int(0)
        rc = ctx.lib.lc_debug_codebook(ctx.h, hist.ctypes.data, nb, lengths.ctypes.data, codes.ctypes.data,
                                       ctypes.byref(ml))
        assert rc == 0, nm
        assert np.array_equal(lengths[:f.size], want), nm
        assert not lengths[f.size:].any()
        used = want > 0
        if used.any():
            assert np.array_equal(codes[:f.size][used], orc.canonical_codes(want)[used]), nm
        deepest = max(deepest, ml.value)
    assert deepest == 39


def test_edge_corpus_relaunches_reported(lc, ctx):
    """The adversarial corpus makes guess-chain decisions differ from the reference's
    (margins of a few ulps): every difference is caught and repaired (relaunches, then
    the sequential chain), and the stats report it."""
    x = _edge(200_000)
    ref = orc.to_bytes(orc.compress(x, "absolute", 1e-3))
    blk = lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.absolute(1e-3))
    assert blk.to_bytes() == ref
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_RESUME, 0)          # the same through full relaunches
    assert lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.absolute(1e-3)).to_bytes() == ref
    ctx.lib.lc_ctx_set_option(ctx.h, OPT_RESUME, 1)
    blk = lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.absolute(1e-3))
    assert ctx.lib.lc_ctx_get_stat(ctx.h, STAT_QUANT_RELAUNCHES) >= 1
    assert ctx.lib.lc_ctx_get_stat(ctx.h, 4) >= 1                          # chunks re-run exactly


def test_subnormal_ulp_vectors(lc, ctx):
    """Vectors whose values are so small that their ulps are subnormal (|x| < 2^-960): the
    offset-map arithmetic is not exact there, so the quantizer certifies nothing and falls back
    to exact re-runs / the sequential chain.  Bytes equal the oracle's, v3 tables and both
    reconstructions are exact (found by a randomized run: v3 sync starts were off by an ulp)."""
    r = np.random.default_rng(5)
    for n, sc, eb in ((4098, 1e-300, 1e-2), (50_000, 1e-300, 1e-4), (300_000, 1e-305, 1e-3), (300_000, 1e-290, 1e-5)):
        x = r.normal(0, sc, n).cumsum()
        ref = orc.compress(x, "value_range_relative", eb)
        b1 = lc.compress(x, lc.CompressorConfig.value_range_relative(eb))
        assert b1.to_bytes() == orc.to_bytes(ref), (n, sc, eb)
        b3 = lc.compress(x, lc.CompressorConfig.value_range_relative(eb, block_version=3))
        st, es = orc.sync_v3(ref["codes"], ref["recon"])
        assert np.array_equal(b3.sync_starts.view(np.int64), st.view(np.int64)), (n, sc, eb)
        for b in (b1, b3):
            assert np.array_equal(lc.decompress(b).view(np.int64), ref["recon"].view(np.int64)), (n, sc, eb, b.version)
    n = 400_000                                                # decays into the subnormal range and back
    env = np.concatenate([np.logspace(0, -320, n // 2), np.logspace(-320, 0, n // 2)])
    x = env * (1 + 0.1 * np.sin(np.arange(n) / 50.0))
    ref = orc.compress(x, "absolute", 1e-293)
    for v in (1, 3):
        b = lc.compress(x, lc.CompressorConfig.absolute(1e-293, block_version=v))
        assert np.array_equal(lc.decompress(b).view(np.int64), ref["recon"].view(np.int64)), v
    assert lc.compress(x, lc.CompressorConfig.absolute(1e-293)).to_bytes() == orc.to_bytes(ref)


def test_small_bin_budgets_v3_tables(lc, ctx):
    """n_bins_half = 1 / 7 with an error bound comparable to the data: the chain cannot follow x and
    sits far from the guess lattice, so the offsets are not exactly representable (a randomized run
    found v3 sync starts off by an ulp).  Such budgets are never certified: tables, bytes and
    both reconstructions are exact."""
    r = np.random.default_rng(3)
    n = 300_000
    t = np.arange(n) / n
    mixed = np.sin(40 * t) * (1 + 1e3 * (r.random(n) < 1e-4)) + r.normal(0, 1e-4, n)
    steps = np.repeat(r.normal(0, 1, 10_000), 100)[:999_999].copy()
    for x, frac, nbh in ((mixed, 0.011, 1), (mixed, 0.011, 7), (steps, 0.0088, 1), (r.normal(0, 1, 49_999), 0.019, 1)):
        eb = frac * float(np.ptp(x))
        ref = orc.compress(x, "absolute", eb, n_bins_half=nbh)
        b1 = lc.compress(x, lc.CompressorConfig.absolute(eb, n_bins_half=nbh))
        assert b1.to_bytes() == orc.to_bytes(ref), (x.size, nbh)
        b3 = lc.compress(x, lc.CompressorConfig.absolute(eb, n_bins_half=nbh, block_version=3))
        st, es = orc.sync_v3(ref["codes"], ref["recon"])
        assert np.array_equal(b3.sync_starts.view(np.int64), st.view(np.int64)), (x.size, nbh)
        for b in (b1, b3):
            assert np.array_equal(lc.decompress(b).view(np.int64), ref["recon"].view(np.int64)), (x.size, nbh, b.version)
