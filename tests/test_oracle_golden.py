"""Pin the CPU oracle (oracle/) against golden vectors from the real reference.

tests/golden/golden.npz was produced by tests/golden/make_golden.py running the
unmodified reference (lossyckpt).  Every oracle output must match bit for bit:
serialized blocks, reconstructions, Huffman code lengths and decode statuses.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import MODES, golden_block_names


def _cases(z):
    return golden_block_names(z)


def test_golden_blocks_match_reference(golden):
    z = golden
    names = _cases(z)
    assert len(names) > 150
    for name in names:
        x = z[str(z[f"{name}/x"])]
        mode, param, nbh = z[f"{name}/cfg"]
        blk = orc.compress(x, MODES[int(mode)], float(param), int(nbh))
        ref = z[f"{name}/block"].tobytes()
        assert orc.to_bytes(blk) == ref, name
        # decompress the reference's own bytes with the oracle
        parsed = orc.from_bytes(ref)
        rec = orc.decompress(parsed)
        assert hashlib.sha256(rec.tobytes()).hexdigest() == str(z[f"{name}/recon_sha256"]), name
        if parsed["payload_bits"]:
            codes = orc.decode(parsed["payload"], parsed["payload_bits"], parsed["code_lengths"],
                               parsed["n"] - 1)
            assert np.array_equal(codes, blk["codes"]), name


def test_golden_huffman_lengths(golden):
    z = golden
    names = sorted({k.split("/")[0] for k in z.files if k.startswith("huff_")})
    assert len(names) >= 80
    for name in names:
        got = orc.code_lengths(z[f"{name}/freqs"])
        assert np.array_equal(got, z[f"{name}/lengths"]), name


def test_golden_decode_statuses(golden):
    z = golden
    names = sorted({k.split("/")[0] for k in z.files if k.startswith("derr_")})
    assert len(names) == 40
    for name in names:
        bits, count = (int(v) for v in z[f"{name}/bits"])
        payload = z[f"{name}/payload"].tobytes()
        want = str(z[f"{name}/status"])
        try:
            out = orc.decode(payload, bits, z[f"{name}/lengths"], count)
            got = "ok"
            assert np.array_equal(out, z[f"{name}/out"]), name
        except orc.OracleIntegrityError as e:
            got = str(e)
        assert got == want, name


def test_known_answer_huffman():
    # huffman tests: test_canonical_codes_frozen_case (test_huffman.py:31-35)
    lengths = orc.code_lengths(np.array([1, 1, 2]))
    assert list(lengths) == [2, 2, 1]
    assert list(orc.canonical_codes(lengths)) == [0b10, 0b11, 0]
    # all-identical symbols pack to one bit each (test_huffman.py:17-21)
    sym = np.full(1000, 7)
    lengths = orc.code_lengths(np.bincount(sym, minlength=8))
    payload, bits = orc.encode(sym, lengths)
    assert bits == 1000
    assert np.array_equal(orc.decode(payload, bits, lengths, 1000), sym)


def test_oracle_rejects_like_reference():
    with pytest.raises(orc.OracleParameterError):
        orc.compress(np.array([]), "absolute", 1.0)
    with pytest.raises(orc.OracleParameterError):
        orc.compress(np.array([1.0, np.inf]), "absolute", 1.0)
    with pytest.raises(orc.OracleIntegrityError):
        orc.from_bytes(b"WRONG!!!" + bytes(64))


def test_oracle_matches_reference_stress_hashes():
    """The oracle on the large stress corpora (tests/stress_inputs.py, <= 2^21 elements
    here to keep the CPU suite short) reproduces the real reference's block and
    reconstruction hashes (tests/golden/stress_golden.json)."""
    import hashlib
    import json
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    import stress_inputs
    gold = json.load(open(os.path.join(here, "golden", "stress_golden.json")))
    checked = 0
    for name, gen, mode, eb, nbh in stress_inputs.CASES:
        g = gold[name]
        if g["n"] > (1 << 21):
            continue
        x = gen()
        assert hashlib.sha256(x.tobytes()).hexdigest() == g["x_sha256"], name
        d = orc.compress(x, mode, eb, n_bins_half=nbh)
        assert hashlib.sha256(orc.to_bytes(d)).hexdigest() == g["block_sha256"], name
        assert hashlib.sha256(d["recon"].tobytes()).hexdigest() == g["recon_sha256"], name
        checked += 1
    assert checked >= 4
