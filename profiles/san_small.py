"""Small compress/decompress round trips (v1, v2, v3; relative and absolute; escapes)
for compute-sanitizer runs."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1805_07384_b200 as lc
from oracle import oracle as orc
r = np.random.default_rng(1)
xs = [np.cumsum(r.normal(size=20000)), np.sin(np.arange(50000) / 300.0) + r.normal(0, 1e-3, 50000)]
xs[0][[5, 777, 19000]] += 1e6
for x in xs:
    for eb in (1e-3, 1e-6):
        ref = orc.compress(x, "value_range_relative", eb)
        for v in (1, 2, 3):
            blk = lc.compress(torch.from_numpy(x).cuda(), lc.CompressorConfig.value_range_relative(eb, block_version=v))
            rec = lc.decompress(lc.CompressedBlock.from_bytes(blk.to_bytes()))
            assert np.array_equal(rec.view(np.int64), ref["recon"].view(np.int64)), (v, eb)
from paper_1805_07384_b200 import solvers
a = solvers.generate_laplacian3d(32)
s = solvers.init("cg", a, solvers.jacobi_preconditioner(a), torch.from_numpy(r.uniform(-1, 1, a.n_rows)).cuda(),
                 solvers.SolveConfig(tolerance=1e-8, restart_len=10))
s.advance(25)
blk = lc.compress(s.x, lc.CompressorConfig.value_range_relative(1e-5, block_version=3), value_range=s.x_range)
lc.decompress(blk, device="cuda")
g = solvers.init("gmres", solvers.generate_convdiff3d(16), solvers.jacobi_preconditioner(solvers.generate_convdiff3d(16)),
                 torch.ones(16 ** 3, dtype=torch.float64).cuda(), solvers.SolveConfig(tolerance=1e-8, restart_len=6))
g.advance(14)
print("sanitizer workload ok")
