"""Profiling driver: one warm-up + one measured compress/decompress of the config-2 vector
(n = 2^26) at one bound through the public API.  Used under ncu:

    python profiles/prof_codec.py [eb_rel] [log2n] [block_version]
Prints the quantizer's relaunches and exactly re-run chunks of the last compress.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_07384_b200 as lc  # noqa: E402
from paper_1805_07384_b200 import _native  # noqa: E402
from bench import make_vector  # noqa: E402

eb = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 26)
xd = torch.from_numpy(make_vector(n)).cuda()
ver = int(sys.argv[3]) if len(sys.argv) > 3 else 1          # block version (3: one-pass decoder)
cfg = lc.CompressorConfig.value_range_relative(eb)
for _ in range(2):
    blk = lc.compress(xd, cfg, block_version=ver)
    rec = lc.decompress(blk, device="cuda")
torch.cuda.synchronize()
err = float((rec - xd).abs().max())
assert err <= blk.eb_abs, (err, blk.eb_abs)
ctx = _native.context(0)
print("ok", n, eb, blk.payload_bits, err / blk.eb_abs, "relaunches", ctx.lib.lc_ctx_get_stat(ctx.h, 0),
      "exact_chunks", ctx.lib.lc_ctx_get_stat(ctx.h, 4))
