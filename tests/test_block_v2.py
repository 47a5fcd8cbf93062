"""Block format v2: LCKP0001 version 2 adds a table
of payload bit offsets every SYNC_K = 1024 symbols, so the decoder starts
every thread at a known codeword boundary (no segment synchronisation).

Bars: the sync table equals the oracle's prefix sums of code lengths; a v2
block's codes, payload and escapes are the v1 block's (bit-exact to the
reference); v2 reconstruction is bit-identical to v1/the oracle; a sync table
that disagrees with the payload raises IntegrityError (status 6)."""

import dataclasses

import numpy as np
import pytest

from oracle import oracle as orc


def _blk(lc, x, eb_rel, version):
    return lc.compress(x, lc.CompressorConfig.value_range_relative(eb_rel, block_version=version))


def test_v2_wire_format_roundtrip_cpu():
    """to_bytes/from_bytes of a v2 block assembled from the oracle (no GPU)."""
    import paper_1805_07384_b200 as lc
    x = np.random.default_rng(2).normal(size=5000).cumsum()
    ref = orc.compress(x, "value_range_relative", 1e-5)
    sync = orc.sync_offsets(ref["codes"], ref["code_lengths"])
    assert sync.size == -(-(x.size - 1) // 1024)
    blk = lc.CompressedBlock(n=ref["n"], eb_abs=ref["eb_abs"], value_range=ref["value_range"],
                             first_value=ref["first_value"], code_lengths=ref["code_lengths"],
                             payload=ref["payload"], payload_bits=ref["payload_bits"],
                             escape_indices=ref["escape_indices"], escape_values=ref["escape_values"],
                             version=2, sync_offsets=sync)
    raw = blk.to_bytes()
    v1 = orc.to_bytes(ref)
    assert len(raw) == len(v1) + 12 + 8 * sync.size
    back = lc.CompressedBlock.from_bytes(raw)
    assert back.version == 2 and np.array_equal(back.sync_offsets, sync)
    assert back.payload == ref["payload"] and back.to_bytes() == raw
    bad = bytearray(raw)
    off = len(v1) - len(ref["payload"])             # sync_k field follows payload_bits
    bad[off:off + 4] = (512).to_bytes(4, "little")
    with pytest.raises(lc.IntegrityError):
        lc.CompressedBlock.from_bytes(bytes(bad))
    with pytest.raises(lc.IntegrityError):
        lc.CompressedBlock.from_bytes(raw[:off + 20])
    with pytest.raises(lc.ParameterError):
        lc.CompressorConfig.absolute(1.0, block_version=4)


def test_v3_wire_format_roundtrip_cpu():
    """v3 = v2 + the chain value and escape count at every sync point (oracle-built)."""
    import paper_1805_07384_b200 as lc
    x = np.random.default_rng(3).normal(size=7000).cumsum()
    x[[10, 2500, 6999]] += 1e6
    ref = orc.compress(x, "value_range_relative", 1e-5)
    sync = orc.sync_offsets(ref["codes"], ref["code_lengths"])
    starts, escs = orc.sync_v3(ref["codes"], ref["recon"])
    assert starts[0] == x[0] and escs[0] == 0 and escs[-1] <= len(ref["escape_indices"])
    blk = lc.CompressedBlock(n=ref["n"], eb_abs=ref["eb_abs"], value_range=ref["value_range"],
                             first_value=ref["first_value"], code_lengths=ref["code_lengths"],
                             payload=ref["payload"], payload_bits=ref["payload_bits"],
                             escape_indices=ref["escape_indices"], escape_values=ref["escape_values"],
                             version=3, sync_offsets=sync, sync_starts=starts, sync_escapes=escs)
    raw = blk.to_bytes()
    assert len(raw) == len(orc.to_bytes(ref)) + 12 + 24 * sync.size
    back = lc.CompressedBlock.from_bytes(raw)
    assert back.version == 3 and back.to_bytes() == raw
    assert np.array_equal(back.sync_starts.view(np.int64), starts.view(np.int64))
    assert np.array_equal(back.sync_escapes, escs)
    with pytest.raises(lc.IntegrityError):
        lc.CompressedBlock.from_bytes(raw[:len(raw) - len(ref["payload"]) - 8])


torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_07384_b200 as lc
    return lc


def _sine(n, seed=0):
    r = np.random.default_rng(seed)
    t = np.arange(n) / n
    out = sum(r.uniform(0, 1) * np.sin(2 * np.pi * r.uniform(1, 64) * t + r.uniform(0, 6)) for _ in range(8))
    return out + r.normal(0, 1e-3, n)


@pytest.mark.gpu
def test_v2_matches_v1_and_oracle(lc):
    rng = np.random.default_rng(77)
    cases = [(_sine(200_001, 1), 1e-4), (rng.normal(size=70_000).cumsum(), 1e-7),
             (rng.normal(size=1025), 1e-2), (rng.normal(size=1024), 1e-3), (rng.normal(size=2), 1e-3)]
    spiky = rng.normal(size=30_000).cumsum()
    spiky[rng.integers(0, spiky.size, 5)] += 1e9
    cases.append((spiky, 1e-9))
    for x, eb in cases:
        b1 = _blk(lc, x, eb, 1)
        b2 = _blk(lc, x, eb, 2)
        ref = orc.compress(x, "value_range_relative", eb)
        assert b2.payload == b1.payload and np.array_equal(b2.escape_indices, b1.escape_indices)
        assert np.array_equal(b2.sync_offsets, orc.sync_offsets(ref["codes"], ref["code_lengths"]))
        b2 = lc.CompressedBlock.from_bytes(b2.to_bytes())
        r2 = lc.decompress(b2)
        assert np.array_equal(r2.view(np.int64), ref["recon"].view(np.int64)), (x.size, eb)
        assert np.array_equal(r2.view(np.int64), lc.decompress(b1).view(np.int64))


@pytest.mark.gpu
def test_v2_full_size(lc):
    n = 1 << 26
    x = _sine(n, 5)
    b2 = _blk(lc, x, 1e-6, 2)
    b1 = _blk(lc, x, 1e-6, 1)
    assert b2.sync_offsets.size == -(-(n - 1) // 1024)
    assert np.all(np.diff(b2.sync_offsets.astype(np.int64)) > 0)
    d2 = lc.decompress(b2, device="cuda")
    d1 = lc.decompress(b1, device="cuda")
    assert torch.equal(d1.view(torch.int64), d2.view(torch.int64))
    assert float((d2 - torch.from_numpy(x).cuda()).abs().max()) <= b2.eb_abs


@pytest.mark.gpu
def test_v2_corrupted_sync_table(lc):
    x = np.random.default_rng(4).normal(size=50_000).cumsum()
    b2 = _blk(lc, x, 1e-6, 2)
    for j, delta in ((1, 1), (3, -1), (b2.sync_offsets.size - 1, 5), (0, 1)):
        s = b2.sync_offsets.copy()
        s[j] = np.uint64(int(s[j]) + delta)
        with pytest.raises(lc.IntegrityError):
            lc.decompress(dataclasses.replace(b2, sync_offsets=s))
    s = b2.sync_offsets.copy()
    s[2] = np.uint64(b2.payload_bits + 100)
    with pytest.raises(lc.IntegrityError):
        lc.decompress(dataclasses.replace(b2, sync_offsets=s))
    with pytest.raises(lc.IntegrityError):
        lc.decompress(dataclasses.replace(b2, sync_offsets=b2.sync_offsets[:-1]))


@pytest.mark.gpu
def test_v3_tables_and_reconstruction(lc):
    """v3 blocks: codes/payload/escapes are v1's (the reference's); the sync tables
    equal the oracle's (bit offsets, reconstruction values, escape counts); the
    one-pass v3 decoder reconstructs bit-identically to the reference."""
    rng = np.random.default_rng(78)
    spiky = rng.normal(size=30_000).cumsum()
    spiky[rng.integers(0, spiky.size, 5)] += 1e9
    cases = [(_sine(200_001, 1), 1e-4), (rng.normal(size=70_000).cumsum(), 1e-7),
             (rng.normal(size=1025), 1e-2), (rng.normal(size=1024), 1e-3), (rng.normal(size=2), 1e-3),
             (spiky, 1e-9), (_sine(100_000, 2), 1e-3)]
    for x, eb in cases:
        b1 = _blk(lc, x, eb, 1)
        b3 = _blk(lc, x, eb, 3)
        ref = orc.compress(x, "value_range_relative", eb)
        assert b3.payload == b1.payload and np.array_equal(b3.escape_indices, b1.escape_indices)
        st, es = orc.sync_v3(ref["codes"], ref["recon"])
        assert np.array_equal(b3.sync_offsets, orc.sync_offsets(ref["codes"], ref["code_lengths"]))
        assert np.array_equal(b3.sync_starts.view(np.int64), st.view(np.int64)), (x.size, eb)
        assert np.array_equal(b3.sync_escapes, es)
        b3 = lc.CompressedBlock.from_bytes(b3.to_bytes())
        r3 = lc.decompress(b3)
        assert np.array_equal(r3.view(np.int64), ref["recon"].view(np.int64)), (x.size, eb)


@pytest.mark.gpu
def test_v3_full_size_and_relaunch_paths(lc):
    """2^26 elements at 1e-6 (v3 decode == v1 decode), and v3 tables through the
    quantizer's resume / full-relaunch / sequential paths (injected failure)."""
    from paper_1805_07384_b200 import _native
    n = 1 << 26
    x = _sine(n, 5)
    b3 = _blk(lc, x, 1e-6, 3)
    b1 = _blk(lc, x, 1e-6, 1)
    d1 = lc.decompress(b1, device="cuda")
    d3 = lc.decompress(b3, device="cuda")
    assert torch.equal(d1.view(torch.int64), d3.view(torch.int64))
    assert torch.equal(torch.from_numpy(b3.sync_starts).cuda().view(torch.int64), d1[:n - 1:1024].view(torch.int64))
    ctx = _native.context(0)
    y = _sine(300_000, 6)
    ref = orc.compress(y, "absolute", 1e-3)
    st, es = orc.sync_v3(ref["codes"], ref["recon"])
    try:
        for resume, maxr in ((1, 64), (0, 64), (1, 0)):
            ctx.lib.lc_ctx_set_option(ctx.h, 5, resume)
            ctx.lib.lc_ctx_set_option(ctx.h, 0, maxr)
            ctx.lib.lc_ctx_set_option(ctx.h, 4, 1)
            ctx.lib.lc_ctx_set_option(ctx.h, 2, 5000)           # wrong prediction for chunk 5000
            b = lc.compress(y, lc.CompressorConfig.absolute(1e-3, block_version=3))
            assert ctx.lib.lc_ctx_get_stat(ctx.h, 0) == 1
            assert np.array_equal(b.sync_starts.view(np.int64), st.view(np.int64)), (resume, maxr)
            assert np.array_equal(b.sync_escapes, es)
            assert np.array_equal(lc.decompress(b).view(np.int64), ref["recon"].view(np.int64))
    finally:
        for k, v in ((5, 1), (0, 64), (4, 0), (2, -1)):
            ctx.lib.lc_ctx_set_option(ctx.h, k, v)


@pytest.mark.gpu
def test_v3_corrupted_tables(lc):
    x = np.random.default_rng(4).normal(size=50_000).cumsum()
    x[[100, 20_000]] += 1e7
    b3 = _blk(lc, x, 1e-6, 3)
    assert lc.decompress(b3).size == x.size
    for field, j, f in (("sync_starts", 1, lambda v: np.nextafter(v, np.inf)),
                        ("sync_starts", 0, lambda v: v + 1.0),
                        ("sync_starts", b3.sync_starts.size - 1, lambda v: -v),
                        ("sync_escapes", 30, lambda v: v + np.uint64(1)),
                        ("sync_offsets", 5, lambda v: v + np.uint64(1))):
        t = getattr(b3, field).copy()
        t[j] = f(t[j])
        with pytest.raises(lc.IntegrityError):
            lc.decompress(dataclasses.replace(b3, **{field: t}))
    with pytest.raises(lc.IntegrityError):
        lc.decompress(dataclasses.replace(b3, escape_indices=b3.escape_indices + 1))


@pytest.mark.gpu
def test_v3_straight_line_walk_variants(lc):
    """The v3 decoder's straight-line walk in its four specialisations and its fallbacks:
    long codes (13..32 bits) with u16 symbols (16-bit prefix symbol table) and with u32 symbols
    (bin budget 100000: the table is unusable), escapes in most intervals, escape-free tiny
    alphabets, a short last interval, vectors shorter than one warp group -- all bit-identical
    to the reference reconstruction and equal to the v1 decode."""
    rng = np.random.default_rng(81)
    walk = rng.normal(size=600_000).cumsum()
    spiky = walk.copy()
    spiky[rng.integers(0, spiky.size, 6000)] += 1e8                    # escapes in most intervals
    cases = [(walk, dict(eb=1e-7), {}),                                  # long codes, u16 symbols
             (walk, dict(eb=1e-7), dict(n_bins_half=100_000)),           # long codes, u32 symbols
             (spiky, dict(eb=1e-9), {}),                                 # escapes + long codes
             (_sine(300_000, 3) , dict(eb=1e-2), {}),                    # tiny alphabet, no escapes
             (spiky[:40_000], dict(eb=1e-3), {}),                        # escapes, short codes
             (walk[:1500], dict(eb=1e-5), {}), (walk[:33 * 1024 + 7], dict(eb=1e-5), {})]
    for x, kw, ckw in cases:
        cfg3 = lc.CompressorConfig.value_range_relative(kw["eb"], block_version=3, **ckw)
        b3 = lc.compress(x, cfg3)
        ref = orc.compress(x, "value_range_relative", kw["eb"], n_bins_half=ckw.get("n_bins_half", 32768))
        r3 = lc.decompress(lc.CompressedBlock.from_bytes(b3.to_bytes()))
        assert np.array_equal(r3.view(np.int64), ref["recon"].view(np.int64)), (x.size, kw, ckw)
        b1 = lc.compress(x, lc.CompressorConfig.value_range_relative(kw["eb"], **ckw))
        assert np.array_equal(lc.decompress(b1).view(np.int64), r3.view(np.int64))
