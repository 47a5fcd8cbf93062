"""CPU oracle for the lossy-checkpoint compressor -- TEST INFRASTRUCTURE ONLY.

Python glue over oracle/lc_oracle.c (a C restatement of the reference's numba
kernels) plus numpy restatements of the reference's host-side steps.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this module; the product package (paper_1805_07384_b200) never does.

Reference: /root/reference/pkg/src/lossyckpt/{compressor,huffman}.py
(file:line cited per function).  Pinned against golden vectors produced by
the real reference: tests/golden/make_golden.py, tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liblc_oracle.so")
_lib = None

BLOCK_MAGIC = b"LCKP0001"
BLOCK_VERSION = 1

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)


class OracleIntegrityError(RuntimeError):
    pass


class OracleParameterError(ValueError):
    pass


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.lco_compress_kernel.restype = ctypes.c_int64
        L.lco_compress_kernel.argtypes = [_f64p, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                          ctypes.c_int, _i64p, _f64p, _f64p, _f64p, _i64p]
        L.lco_decompress_kernel.restype = ctypes.c_int64
        L.lco_decompress_kernel.argtypes = [_i64p, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                            _f64p, ctypes.c_int64, _f64p]
        L.lco_code_lengths.restype = ctypes.c_int
        L.lco_code_lengths.argtypes = [_i64p, ctypes.c_int64, _u8p]
        L.lco_canonical_codes.restype = ctypes.c_int
        L.lco_canonical_codes.argtypes = [_u8p, ctypes.c_int64, _u64p]
        L.lco_encode_kernel.restype = ctypes.c_uint64
        L.lco_encode_kernel.argtypes = [_i64p, ctypes.c_int64, _u64p, _u8p, _u8p]
        L.lco_decode_kernel.restype = ctypes.c_int
        L.lco_decode_kernel.argtypes = [_u8p, ctypes.c_uint64, _u8p, ctypes.c_int64,
                                        ctypes.c_int64, _i64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


# --- kernels ---------------------------------------------------------------

def compress_kernel(data, eb_abs, n_bins_half=32768, record=False):
    """compressor.py:319-355 -> (codes i64[n-1], recon f64[n], esc_idx i64[], pe, pe_rec)."""
    data = np.ascontiguousarray(data, dtype=np.float64)
    n = data.size
    codes = np.empty(max(n - 1, 1), dtype=np.int64)
    recon = np.empty(n, dtype=np.float64)
    tl = n - 1 if record else 1
    pe = np.empty(max(tl, 1), dtype=np.float64)
    pe_rec = np.empty(max(tl, 1), dtype=np.float64)
    esc = np.empty(n, dtype=np.int64)
    k = lib().lco_compress_kernel(_p(data, _f64p), n, float(eb_abs), int(n_bins_half), int(record),
                                  _p(codes, _i64p), _p(recon, _f64p), _p(pe, _f64p),
                                  _p(pe_rec, _f64p), _p(esc, _i64p))
    return codes[: n - 1], recon, esc[:k].copy(), pe[:tl], pe_rec[:tl]


def decompress_kernel(codes, n, first_value, delta, escape_values):
    """compressor.py:358-376 -> (out f64[n], escapes used or -1)."""
    codes = np.ascontiguousarray(codes, dtype=np.int64)
    ev = np.ascontiguousarray(escape_values, dtype=np.float64)
    out = np.empty(n, dtype=np.float64)
    evp = ev if ev.size else np.zeros(1)
    used = lib().lco_decompress_kernel(_p(codes if codes.size else np.zeros(1, np.int64), _i64p), n,
                                       float(first_value), float(delta), _p(evp, _f64p), ev.size,
                                       _p(out, _f64p))
    return out, used


def code_lengths(freqs):
    """huffman.py:21-55."""
    freqs = np.ascontiguousarray(freqs, dtype=np.int64)
    out = np.zeros(freqs.size, dtype=np.uint8)
    if freqs.size == 0:
        return out
    if lib().lco_code_lengths(_p(freqs, _i64p), freqs.size, _p(out, _u8p)) != 0:
        raise OracleParameterError("frequencies must be non-negative")
    return out


def canonical_codes(lengths):
    """huffman.py:58-72."""
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    out = np.zeros(lengths.size, dtype=np.uint64)
    if lengths.size and lib().lco_canonical_codes(_p(lengths, _u8p), lengths.size, _p(out, _u64p)):
        raise OracleParameterError("code length exceeds 64 bits")
    return out


def encode(symbols, lengths):
    """huffman.py:135-150 -> (payload bytes, bits)."""
    symbols = np.ascontiguousarray(symbols, dtype=np.int64)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    if symbols.size == 0:
        return b"", 0
    if symbols.min() < 0 or symbols.max() >= len(lengths):
        raise OracleParameterError("symbol outside the codebook alphabet")
    per = lengths[symbols].astype(np.int64)
    if np.any(per == 0):
        raise OracleParameterError("symbol with zero frequency cannot be encoded")
    total = int(per.sum())
    out = np.zeros((total + 7) // 8, dtype=np.uint8)
    codes = canonical_codes(lengths)
    written = lib().lco_encode_kernel(_p(symbols, _i64p), symbols.size, _p(codes, _u64p),
                                      _p(lengths, _u8p), _p(out if out.size else np.zeros(1, np.uint8), _u8p))
    assert written == total
    return out.tobytes(), total


DECODE_REASONS = {1: "invalid codeword", 2: "payload exhausted mid-symbol",
                  3: "trailing bits after last symbol"}


def decode_status(payload, bit_length, lengths, count):
    """huffman.py:153-172; returns (status, symbols).  status: 0 ok, 1/2/3 as the
    reference's _decode_kernel, or a string for the pre-kernel IntegrityErrors."""
    if count == 0:
        if bit_length != 0:
            return "payload bits present but zero symbols expected", None
        return 0, np.zeros(0, dtype=np.int64)
    if bit_length > 8 * len(payload):
        return "payload shorter than its declared bit length", None
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    if not np.any(lengths > 0):
        return "empty codebook cannot decode symbols", None
    buf = np.frombuffer(payload, dtype=np.uint8).copy() if len(payload) else np.zeros(1, np.uint8)
    out = np.empty(count, dtype=np.int64)
    st = lib().lco_decode_kernel(_p(buf, _u8p), int(bit_length), _p(lengths, _u8p), lengths.size,
                                 int(count), _p(out, _i64p))
    return st, out


def decode(payload, bit_length, lengths, count):
    st, out = decode_status(payload, bit_length, lengths, count)
    if isinstance(st, str):
        raise OracleIntegrityError(st)
    if st != 0:
        raise OracleIntegrityError(f"Huffman decode failed: {DECODE_REASONS[st]}")
    return out


# --- full pipeline (compressor.py:379-440) ---------------------------------

def resolve_eb(mode, param, vr):
    """compressor.py:138-148 (+ bound_from_target_psnr 46-50)."""
    if mode == "absolute":
        return float(param)
    if mode == "value_range_relative":
        return float(param) * vr
    if mode == "fixed_psnr":
        return (math.sqrt(3.0) * 10.0 ** (-float(param) / 20.0)) * vr
    raise OracleParameterError(mode)


def compress(data, mode, param, n_bins_half=32768, record=False):
    """compressor.py:379-417.  Returns a dict with the CompressedBlock fields."""
    data = np.ascontiguousarray(data, dtype=np.float64)
    if data.size < 1:
        raise OracleParameterError("cannot compress an empty vector")
    if not np.all(np.isfinite(data)):
        raise OracleParameterError("input contains NaN or Inf")
    vr = float(data.max() - data.min())
    eb = resolve_eb(mode, param, vr)
    if vr == 0.0 or data.size == 1:
        e = np.zeros(0)
        return dict(n=int(data.size), eb_abs=eb, value_range=vr, first_value=float(data[0]),
                    code_lengths=np.zeros(0, np.uint8), payload=b"", payload_bits=0,
                    escape_indices=np.zeros(0, np.int64), escape_values=e,
                    codes=np.zeros(0, np.int64), traces=(e, e) if record else None)
    if not math.isfinite(2.0 * eb):
        raise OracleParameterError("error bound too large to quantize")
    codes, recon, esc, pe, pe_rec = compress_kernel(data, eb, n_bins_half, record)
    freqs = np.bincount(codes, minlength=2 * n_bins_half)
    lengths = code_lengths(freqs)
    payload, bits = encode(codes, lengths)
    return dict(n=int(data.size), eb_abs=eb, value_range=vr, first_value=float(data[0]),
                code_lengths=lengths, payload=payload, payload_bits=bits,
                escape_indices=esc, escape_values=data[esc].copy() if esc.size else np.zeros(0),
                codes=codes, recon=recon, traces=(pe, pe_rec) if record else None)


def sync_offsets(codes, lengths, k=1024):
    """v2 block sync table (no reference counterpart):
    bit offset in the payload of symbol 0, k, 2k, ... (prefix sums of the
    code lengths encode() lays down, huffman.py:131-146)."""
    codes = np.asarray(codes, dtype=np.int64)
    if codes.size == 0:
        return np.zeros(0, np.uint64)
    bits = np.asarray(lengths, dtype=np.uint64)[codes]
    start = np.concatenate([[0], np.cumsum(bits)[:-1]]).astype(np.uint64)
    return start[::k].copy()


def sync_v3(codes, recon, k=1024):
    """v3 block tables beside the bit offsets (no reference counterpart): the
    reference reconstruction at every k-th element (the exact chain value
    before symbol k*j, compressor.py:358-376) and the escape codes before
    symbol k*j (code 0, compressor.py:339-341)."""
    codes = np.asarray(codes, dtype=np.int64)
    if codes.size == 0:
        return np.zeros(0), np.zeros(0, np.uint64)
    starts = np.asarray(recon, dtype=np.float64)[:codes.size:k].copy()
    esc = np.concatenate([[0], np.cumsum(codes == 0)[:-1]]).astype(np.uint64)[::k].copy()
    return starts, esc


def decompress(blk):
    """compressor.py:420-440."""
    n = blk["n"]
    if n < 1:
        raise OracleIntegrityError("block declares zero elements")
    if blk["payload_bits"] == 0 and len(blk["code_lengths"]) == 0:
        if len(blk["escape_indices"]):
            raise OracleIntegrityError("constant block cannot carry escapes")
        return np.full(n, blk["first_value"], dtype=np.float64)
    codes = decode(blk["payload"], blk["payload_bits"], blk["code_lengths"], n - 1)
    out, used = decompress_kernel(codes, n, blk["first_value"], 2.0 * blk["eb_abs"],
                                  blk["escape_values"])
    nd = len(blk["escape_indices"])
    if used < 0 or used != nd:
        raise OracleIntegrityError(f"escape count mismatch: codes need {used}, header has {nd}")
    if nd and not np.array_equal(np.flatnonzero(codes == 0) + 1, blk["escape_indices"]):
        raise OracleIntegrityError("escape positions disagree with escape codes")
    return out


def pack_codebook(code_lengths):
    """compressor.py:179-198."""
    cl = np.asarray(code_lengths)
    used = np.flatnonzero(cl > 0)
    if used.size == 0:
        return struct.pack("<I", 0)
    if used.max() >= 1 << 16:
        raise OracleParameterError("code symbol exceeds the 16-bit wire format")
    order = sorted((int(cl[s]), int(s)) for s in used)
    max_len = order[-1][0]
    counts = np.zeros(max_len, dtype="<u2")
    for length, _ in order:
        counts[length - 1] += 1
    blob = struct.pack("<B", max_len) + counts.tobytes()
    blob += np.array([s for _, s in order], dtype="<u2").tobytes()
    return struct.pack("<I", len(blob)) + blob


def to_bytes(blk):
    """compressor.py:251-267."""
    out = bytearray(BLOCK_MAGIC)
    out += struct.pack("<IQddd", BLOCK_VERSION, blk["n"], blk["eb_abs"], blk["value_range"],
                       blk["first_value"])
    out += pack_codebook(blk["code_lengths"])
    out += struct.pack("<Q", len(blk["escape_indices"]))
    for idx, val in zip(blk["escape_indices"], blk["escape_values"]):
        out += struct.pack("<Qd", int(idx), float(val))
    out += struct.pack("<Q", blk["payload_bits"])
    out += blk["payload"]
    return bytes(out)


def _unpack_codebook(blob):
    """compressor.py:201-224."""
    if len(blob) == 0:
        return np.zeros(0, dtype=np.uint8)
    (max_len,) = struct.unpack_from("<B", blob, 0)
    if max_len == 0 or len(blob) < 1 + 2 * max_len:
        raise OracleIntegrityError("malformed codebook header")
    counts = np.frombuffer(blob, dtype="<u2", count=max_len, offset=1)
    n_symbols = int(counts.sum())
    if len(blob) != 1 + 2 * max_len + 2 * n_symbols:
        raise OracleIntegrityError("codebook symbol list disagrees with counts")
    symbols = np.frombuffer(blob, dtype="<u2", offset=1 + 2 * max_len).astype(np.int64)
    lengths = np.zeros(int(symbols.max()) + 1 if n_symbols else 0, dtype=np.uint8)
    pos = 0
    for length in range(1, max_len + 1):
        group = symbols[pos:pos + int(counts[length - 1])]
        if group.size > 1 and np.any(np.diff(group) <= 0):
            raise OracleIntegrityError("codebook symbols not in canonical order")
        if np.any(lengths[group] != 0):
            raise OracleIntegrityError("codebook repeats a symbol")
        lengths[group] = length
        pos += group.size
    return lengths


def from_bytes(blob):
    """compressor.py:269-301 -> block dict."""
    if len(blob) < 8 or blob[:8] != BLOCK_MAGIC:
        raise OracleIntegrityError("not a compressed block (bad magic)")
    off = 8
    try:
        version, n, eb_abs, vr, first_value = struct.unpack_from("<IQddd", blob, off)
        off += struct.calcsize("<IQddd")
        if version != BLOCK_VERSION:
            raise OracleIntegrityError(f"unsupported block version {version}")
        (cb_len,) = struct.unpack_from("<I", blob, off)
        off += 4
        if off + cb_len > len(blob):
            raise OracleIntegrityError("codebook length inconsistent with payload")
        lengths = _unpack_codebook(blob[off:off + cb_len])
        off += cb_len
        (n_esc,) = struct.unpack_from("<Q", blob, off)
        off += 8
        if off + 16 * n_esc > len(blob):
            raise struct.error("escape table truncated")
        pairs = np.frombuffer(blob, dtype=np.dtype([("i", "<u8"), ("v", "<f8")]), count=n_esc, offset=off)
        esc_idx = pairs["i"].astype(np.int64)
        esc_val = pairs["v"].astype(np.float64)
        off += 16 * n_esc
        (payload_bits,) = struct.unpack_from("<Q", blob, off)
        off += 8
    except struct.error as exc:
        raise OracleIntegrityError(f"truncated block: {exc}") from None
    payload = blob[off:]
    if len(payload) != (payload_bits + 7) // 8:
        raise OracleIntegrityError("payload byte count disagrees with bit length")
    return dict(n=n, eb_abs=eb_abs, value_range=vr, first_value=first_value, code_lengths=lengths,
                payload=bytes(payload), payload_bits=payload_bits, escape_indices=esc_idx,
                escape_values=esc_val)
