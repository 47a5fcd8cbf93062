"""Generate solver-harness golden values with the REAL reference (solvers.py,
simulate.measure_n_prime, checkpoint.py, compressor.py).

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_solver_golden.py [--full]

Writes tests/golden/solver_golden.npz with, per case: the grid/stencil, the
rhs, baseline iteration count, N' samples, x after a few Jacobi steps and the
first residual norms.  --full adds BASELINE.json config 1 (Jacobi on
poisson2d(256), b ~ U(-1,1) seed 0, k=10, tol 1e-6, failure at 200).
Stencil matrices are built through the reference's own
SparseMatrixCsr.from_triplets from the CSR arrays of
paper_1805_07384_b200.solvers.StencilMatrix.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from lossyckpt import simulate, solvers  # noqa: E402
from lossyckpt.compressor import CompressorConfig  # noqa: E402
from lossyckpt.sparse import SparseMatrixCsr, jacobi_preconditioner  # noqa: E402

from paper_1805_07384_b200.solvers import StencilMatrix  # noqa: E402  (pure numpy part)

OUT = os.path.join(ROOT, "tests", "golden", "solver_golden.npz")
cases = {}


def csr(st):
    ro, ci, va = st.to_csr_arrays()
    rows = np.repeat(np.arange(st.n_rows), np.diff(ro))
    return SparseMatrixCsr.from_triplets(st.n_rows, st.n_cols, rows, ci, va)


def add(name, st, method, b, cfg, eb_rel, inject=None, jac_steps=0):
    a = csr(st)
    m = jacobi_preconditioner(a)
    base = solvers.solve_to_convergence(solvers.init(method, a, m, b, cfg))
    pts = inject if inject is not None else [base.iteration // 3, (2 * base.iteration) // 3]
    res = simulate.measure_n_prime(method, a, m, b, cfg, CompressorConfig.value_range_relative(eb_rel), pts)
    cases[name + "/stencil"] = np.array([st.nx, st.ny, st.nz, st.c, st.xm, st.xp, st.ym, st.yp, st.zm, st.zp])
    cases[name + "/b"] = b
    cases[name + "/cfg"] = np.array([cfg.tolerance, cfg.max_iterations, cfg.restart_len, cfg.ckpt_intvl, eb_rel])
    cases[name + "/method"] = np.array([["jacobi", "cg", "gmres"].index(method)])
    cases[name + "/baseline"] = np.array([res.baseline_n])
    cases[name + "/inject"] = np.array(pts)
    cases[name + "/nprime"] = res.values()
    s = solvers.init(method, a, m, b, cfg)
    norms = [s.residual_norm]
    for _ in range(12):
        s.step()
        norms.append(s.residual_norm)
    cases[name + "/norms"] = np.array(norms)
    if jac_steps:
        s = solvers.init(method, a, m, b, cfg)
        for _ in range(jac_steps):
            s.step()
        cases[name + "/x_steps"] = s.x.copy()
        cases[name + "/n_steps"] = np.array([jac_steps])
    print(name, "baseline", res.baseline_n, "N'", res.values(), flush=True)


add("jac2d", StencilMatrix(32, 32, 1, 4.0, -1.0, -1.0, -1.0, -1.0),
    "jacobi", np.random.default_rng(0).uniform(-1, 1, 1024),
    solvers.SolveConfig(tolerance=1e-6, max_iterations=10 ** 6, ckpt_intvl=10), 1e-4, [200, 555], jac_steps=100)
add("cg3d", StencilMatrix(10, 10, 10, 6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0),
    "cg", np.random.default_rng(1).uniform(-1, 1, 1000),
    solvers.SolveConfig(tolerance=1e-8, restart_len=20, ckpt_intvl=10), 1e-5)
vx, vy, vz = 0.1, 0.05, 0.025
add("gmres3d", StencilMatrix(8, 8, 8, 6.0 + vx + vy + vz, -1.0 - vx, -1.0, -1.0 - vy, -1.0, -1.0 - vz, -1.0),
    "gmres", np.random.default_rng(2).uniform(-1, 1, 512),
    solvers.SolveConfig(tolerance=1e-8, restart_len=30, ckpt_intvl=10), 1e-4)
if "--full" in sys.argv:
    add("config1", StencilMatrix(256, 256, 1, 4.0, -1.0, -1.0, -1.0, -1.0),
        "jacobi", np.random.default_rng(0).uniform(-1, 1, 65536),
        solvers.SolveConfig(tolerance=1e-6, max_iterations=10 ** 6, ckpt_intvl=10), 1e-4, [200])
np.savez_compressed(OUT, **cases)
print("wrote", OUT)
