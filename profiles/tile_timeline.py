"""Per-tile phase timeline of the single-pass quantizer (LC_TIMELINE=1 diagnostics).

    LC_TIMELINE=1 python profiles/tile_timeline.py [eb_rel] [log2n]
Stamps per tile (globaltimer ns): claim, pass A done (aggregate published),
look-back + exact re-runs done, codes stored; prints phase-time percentiles
and the critical-path shape (claim time and look-back wait versus ticket)."""
import ctypes
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
cfg = lc.CompressorConfig.value_range_relative(eb)
for _ in range(2):
    blk = lc.compress(xd, cfg)
torch.cuda.synchronize()
ctx = _native.context(0)
ntiles = ((n - 1 + 31) // 32 + 255) // 256
buf = np.zeros(ntiles * 16, np.uint64)
ctx.lib.lc_debug_copy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64]
ctx.lib.lc_debug_copy(ctx.h, 6, buf.ctypes.data, buf.nbytes)
tl = buf.reshape(ntiles, 16).astype(np.float64)
t0 = tl[:, 0].min()
claim, a, lb, ex, end = (tl[:, k] - t0 for k in range(5))
print(f"n={n} eb={eb} tiles={ntiles} span {end.max() / 1e3:.1f} us")
for name, v in (("load+passA", a - claim), ("lookback", lb - a), ("exact", ex - lb), ("store", end - ex),
                ("tile total", end - claim)):
    print(f"{name:12s} p10 {np.percentile(v, 10) / 1e3:7.2f} p50 {np.percentile(v, 50) / 1e3:7.2f} "
          f"p90 {np.percentile(v, 90) / 1e3:7.2f} max {v.max() / 1e3:7.2f} us")
for k in range(0, ntiles, max(1, ntiles // 16)):
    print(f"tile {k:6d} claim {claim[k] / 1e3:8.1f} passA {(a[k] - claim[k]) / 1e3:6.2f} "
          f"lookback {(lb[k] - a[k]) / 1e3:6.2f} end {end[k] / 1e3:8.1f} sm {int(tl[k, 6])}")
