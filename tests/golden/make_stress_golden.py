"""Golden hashes for the large stress corpora, from the REAL reference.

Run in the build container (the reference is importable there, not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_stress_golden.py
For each case of tests/stress_inputs.py it records sha256 of the input, of the
reference's CompressedBlock.to_bytes() (compressor.py:251-267) and of decompress()
(compressor.py:420-440), plus block statistics.  Writes tests/golden/stress_golden.json.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from lossyckpt import compressor  # noqa: E402  (the reference)

import stress_inputs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "stress_golden.json")


def sha(b):
    return hashlib.sha256(b).hexdigest()


out = {}
for name, gen, mode, eb, nbh in stress_inputs.CASES:
    x = gen()
    cfg = (compressor.CompressorConfig.absolute(eb, n_bins_half=nbh) if mode == "absolute"
           else compressor.CompressorConfig.value_range_relative(eb, n_bins_half=nbh))
    t0 = time.time()
    blk = compressor.compress(x, cfg)
    data = blk.to_bytes()
    rec = compressor.decompress(blk)
    lengths = np.asarray(blk.code_lengths)
    out[name] = {"mode": mode, "eb": eb, "n_bins_half": nbh, "n": int(x.size), "x_sha256": sha(x.tobytes()),
                 "block_sha256": sha(data), "block_bytes": len(data),
                 "recon_sha256": sha(rec.tobytes()), "n_esc": int(len(blk.escape_indices)),
                 "max_len": int(lengths.max()) if lengths.size else 0,
                 "used_symbols": int((lengths > 0).sum()), "payload_bits": int(blk.payload_bits)}
    print(name, out[name], f"{time.time() - t0:.1f}s", flush=True)
json.dump(out, open(OUT, "w"), indent=1)
print("wrote", OUT)
