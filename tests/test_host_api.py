"""Host-side mirror of the reference API (no GPU): config validation, PSNR
helpers, LCKP0001 wire format, C-ABI exports.  Reference tests mirrored:
test_compressor.py:146-174 (frozen PSNR values), :96-124 (serialization)."""

import ctypes
import math
import re

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1805_07384_b200 import _native
from paper_1805_07384_b200 import compressor as cp
from paper_1805_07384_b200.errors import IntegrityError, ParameterError, UndefinedPsnrError
from tests.conftest import ROOT, golden_block_names


def test_frozen_psnr_values():
    assert cp.estimate_psnr_from_bound(1e-4) == pytest.approx(84.77121254719663, rel=1e-12)
    assert cp.bound_from_target_psnr(80.0) == pytest.approx(1.7320508075688772e-4, rel=1e-12)
    for eb in (1e-6, 1e-4, 1e-2):
        assert cp.bound_from_target_psnr(cp.estimate_psnr_from_bound(eb)) == pytest.approx(eb, rel=1e-12)
    with pytest.raises(ParameterError):
        cp.estimate_psnr_from_bound(0.0)
    with pytest.raises(ParameterError):
        cp.bound_from_target_psnr(-3.0)
    assert cp.psnr_from_bin_width(2e-3 * 2, 2.0) == pytest.approx(cp.estimate_psnr_from_bound(1e-3), rel=1e-12)


def test_mse_helpers():
    assert cp.estimate_mse_general(np.full(5, 0.2), np.full(5, 0.5)) == pytest.approx(0.2 ** 2 / 12, rel=1e-12)
    stats = cp.measured_psnr([0.0, 1.0], [0.5, 0.5])
    assert stats.psnr_db == pytest.approx(6.020599913279624, rel=1e-12)
    assert math.isinf(cp.measured_psnr([0.0, 1.0], [0.0, 1.0]).psnr_db)
    with pytest.raises(UndefinedPsnrError):
        cp.measured_psnr([1.0, 1.0], [1.0, 1.0])


def test_config_validation():
    with pytest.raises(ParameterError):
        cp.CompressorConfig.absolute(0.0)
    with pytest.raises(ParameterError):
        cp.CompressorConfig.absolute(math.inf)
    with pytest.raises(ParameterError):
        cp.CompressorConfig.value_range_relative(1.0)
    with pytest.raises(ParameterError):
        cp.CompressorConfig.fixed_psnr(0.0)
    with pytest.raises(ParameterError):
        cp.CompressorConfig("nope")
    with pytest.raises(ParameterError):
        cp.CompressorConfig.absolute(1.0, n_bins_half=0)
    with pytest.raises(ParameterError):
        cp.CompressorConfig.absolute(1.0, predictor_order=2)
    c = cp.CompressorConfig.fixed_psnr(80.0)
    eb_abs, eb_rel = c.resolve_bounds(2.0)
    assert eb_rel == cp.bound_from_target_psnr(80.0) and eb_abs == eb_rel * 2.0


def test_wire_format_roundtrip_golden(golden):
    """Every golden block parses and re-serialises byte-identically."""
    names = golden_block_names(golden)
    for name in names:
        blob = golden[f"{name}/block"].tobytes()
        blk = cp.CompressedBlock.from_bytes(blob)
        assert blk.to_bytes() == blob, name
        ref = orc.from_bytes(blob)
        assert np.array_equal(blk.code_lengths, ref["code_lengths"])
        assert np.array_equal(blk.escape_indices, ref["escape_indices"])
        assert cp._pack_codebook(ref["code_lengths"]) == orc.pack_codebook(ref["code_lengths"])


def test_wire_format_errors():
    with pytest.raises(IntegrityError, match="bad magic"):
        cp.CompressedBlock.from_bytes(b"WRONG!!!" + bytes(64))
    blk = cp.CompressedBlock(n=5, eb_abs=0.1, value_range=1.0, first_value=0.0,
                             code_lengths=np.array([0, 1, 1], np.uint8), payload=b"\x50",
                             payload_bits=4, escape_indices=np.zeros(0, np.int64),
                             escape_values=np.zeros(0))
    blob = blk.to_bytes()
    for cut in (3, 9, 20):
        with pytest.raises(IntegrityError):
            cp.CompressedBlock.from_bytes(blob[: len(blob) - cut])
    bad_version = blob[:8] + (7).to_bytes(4, "little") + blob[12:]
    with pytest.raises(IntegrityError, match="unsupported block version"):
        cp.CompressedBlock.from_bytes(bad_version)
    with pytest.raises(ParameterError, match="16-bit"):
        cp._pack_codebook(np.r_[np.zeros(70000, np.uint8), [3]])


def test_escape_table_truncation_matches_reference():
    blk = cp.CompressedBlock(n=5, eb_abs=0.1, value_range=1.0, first_value=0.0,
                             code_lengths=np.array([1, 1], np.uint8), payload=b"\x00",
                             payload_bits=4, escape_indices=np.array([1, 2], np.int64),
                             escape_values=np.array([1.0, 2.0]))
    blob = blk.to_bytes()
    cut = blob[: blob.index(b"\x00\x00\xf0?") + 2]
    try:
        orc.from_bytes(cut)
        ref = None
    except orc.OracleIntegrityError as e:
        ref = str(e)
    with pytest.raises(IntegrityError) as ei:
        cp.CompressedBlock.from_bytes(cut)
    assert ref is not None and str(ei.value).split(":")[0] == ref.split(":")[0]


def test_c_abi_exports_every_declared_symbol():
    """The library loads without a GPU and exports every include/*.h entry point."""
    header = open(f"{ROOT}/include/lossyckpt_b200.h").read()
    declared = set(re.findall(r"^\s*(?:int|void|double|uint64_t|long long|const char \*)\s*\**(lc_\w+)\(", header, re.M))
    assert declared >= set(_native.EXPORTED)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for sym in declared:
        assert hasattr(lib, sym), sym
