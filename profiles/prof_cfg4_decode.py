"""Decode timing of BASELINE config 4 state (GMRES iterate of the 256^3 convection-diffusion problem
after 120 iterations) for v1 and v3 blocks at eb_rel 1e-4 and 1e-6 (device ms per decompress)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_07384_b200 as lc
from paper_1805_07384_b200 import _native, solvers
ctx = _native.context(0)
a = solvers.generate_convdiff3d(256)
m = solvers.jacobi_preconditioner(a)
b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, a.n_rows)).cuda()
cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=30, ckpt_intvl=60, max_iterations=100_000)
s = solvers.init("gmres", a, m, b, cfg); s.advance(120)
x = s.x.detach().clone()
for eb in (1e-4, 1e-6):
    for ver in (1, 3):
        blk = lc.compress(x, lc.CompressorConfig.value_range_relative(eb), block_version=ver)
        ts = []
        for _ in range(3):
            rec = lc.decompress(blk, device="cuda"); ts.append(ctx.lib.lc_last_device_ms(ctx.h))
        print("config4 x@120 eb", eb, "v%d" % ver, "decompress device ms", round(min(ts), 3), "esc", len(blk.escape_indices),
              "ok", bool((rec - x).abs().max() <= blk.eb_abs), flush=True)
