"""Golden values for BASELINE.json configs 3 and 4 from the REAL reference
(solvers.py, checkpoint.py, compressor.py), run in the build container:

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_config_golden.py [names...]

Writes tests/golden/config_golden.json: per case the failure-free baseline
iteration count, the final iteration count of a trial with the listed
injected failures (multi_failure_trial below, the protocol the GPU harness's
harness.measure_multi_failure follows), N' = final - baseline, the iterations
recovered from, the compression ratio of every lossy checkpoint taken, and the
first residual norms of a failure-free run.

config3      CG on the 3-D 7-point Laplacian 128^3, b ~ U(-1,1) seed 1,
             tol 1e-8, restart = checkpoint interval = 20, eb_rel 1e-5,
             failures at iterations 100 and 300 (BASELINE.json configs[2]).
config4_*    restarted GMRES(30) on the upwind convection-diffusion stencil,
             b ~ U(-1,1) seed 2, tol 1e-8, checkpoint every 2 cycles (60
             iterations), failure at the end of cycle 5 (iteration 150), eb_rel
             1e-4 and 1e-6 (BASELINE.json configs[3]) -- at 32^3 and 64^3: the 256^3
             problem takes hours per solve on the CPU reference, so the full
             size runs only on the GPU (unpinned there).
Matrices go through the reference's SparseMatrixCsr.from_triplets from the
CSR arrays of paper_1805_07384_b200.solvers.StencilMatrix.
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from lossyckpt import checkpoint as ckpt, solvers  # noqa: E402
from lossyckpt.compressor import CompressorConfig  # noqa: E402
from lossyckpt.sparse import SparseMatrixCsr, jacobi_preconditioner  # noqa: E402

from paper_1805_07384_b200.solvers import generate_convdiff3d, generate_laplacian3d  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "config_golden.json")


def csr(st):
    ro, ci, va = st.to_csr_arrays()
    rows = np.repeat(np.arange(st.n_rows), np.diff(ro))
    return SparseMatrixCsr.from_triplets(st.n_rows, st.n_cols, rows, ci, va)


def multi_failure_trial(method, a, m, b, cfg, comp, failures, k):
    """Run with a lossy checkpoint every k iterations (not re-taken at the
    iteration just recovered to); at each listed iteration (reached for the
    first time) the state is lost and recovered from the last image."""
    store = ckpt.StorageTarget()
    solver = solvers.init(method, a, m, b, cfg)
    pending = sorted(failures)
    last, recovered_at, recs, ratios = None, None, [], []
    while not solver.converged and solver.iteration < cfg.max_iterations:
        it = solver.iteration
        if pending and it == pending[0]:
            pending.pop(0)
            if last is None:
                solver = solvers.init(method, a, m, b, cfg)
            else:
                solver, _ = ckpt.recover(last, method, a, m, b, cfg)
            recs.append(solver.iteration)
            recovered_at = solver.iteration
            continue
        if it > 0 and it % k == 0 and it != recovered_at:
            last, _ = ckpt.checkpoint_lossy(solver, comp, store)
            ratios.append(float(solver.x.nbytes / len(last.payload)))
        solver.step()
    return solver, recs, ratios


CASES = {
    "config3": dict(st=lambda: generate_laplacian3d(128), method="cg", seed=1, tol=1e-8, restart=20, k=20,
                    eb=1e-5, failures=[100, 300]),
    "config4_1e-4": dict(st=lambda: generate_convdiff3d(32), method="gmres", seed=2, tol=1e-8, restart=30, k=60,
                         eb=1e-4, failures=[150]),
    "config4_1e-6": dict(st=lambda: generate_convdiff3d(32), method="gmres", seed=2, tol=1e-8, restart=30, k=60,
                         eb=1e-6, failures=[150]),
    "config4_64_1e-4": dict(st=lambda: generate_convdiff3d(64), method="gmres", seed=2, tol=1e-8, restart=30,
                            k=60, eb=1e-4, failures=[150]),
    "config4_64_1e-6": dict(st=lambda: generate_convdiff3d(64), method="gmres", seed=2, tol=1e-8, restart=30,
                            k=60, eb=1e-6, failures=[150]),
    "config4_128_1e-4": dict(st=lambda: generate_convdiff3d(128), method="gmres", seed=2, tol=1e-8, restart=30,
                             k=60, eb=1e-4, failures=[150]),
    "config4_128_1e-6": dict(st=lambda: generate_convdiff3d(128), method="gmres", seed=2, tol=1e-8, restart=30,
                             k=60, eb=1e-6, failures=[150]),
    "config4_256_1e-4": dict(st=lambda: generate_convdiff3d(256), method="gmres", seed=2, tol=1e-8, restart=30,
                             k=60, eb=1e-4, failures=[150]),
    "config4_256_1e-6": dict(st=lambda: generate_convdiff3d(256), method="gmres", seed=2, tol=1e-8, restart=30,
                             k=60, eb=1e-6, failures=[150]),
}

gold = json.load(open(OUT)) if os.path.exists(OUT) else {}
for name in (sys.argv[1:] or list(CASES)):
    c = CASES[name]
    st = c["st"]()
    a = csr(st)
    m = jacobi_preconditioner(a)
    b = np.random.default_rng(c["seed"]).uniform(-1, 1, st.n_rows)
    cfg = solvers.SolveConfig(tolerance=c["tol"], restart_len=c["restart"], ckpt_intvl=c["k"],
                              max_iterations=100_000)
    t0 = time.time()
    s = solvers.init(c["method"], a, m, b, cfg)
    norms = [s.residual_norm]
    for _ in range(40):
        s.step()
        norms.append(s.residual_norm)
    solvers.solve_to_convergence(s)
    base = s.iteration
    comp = CompressorConfig.value_range_relative(c["eb"])
    fin, recs, ratios = multi_failure_trial(c["method"], a, m, b, cfg, comp, c["failures"], c["k"])
    gold[name] = dict(grid=[st.nx, st.ny, st.nz], stencil=[st.c, st.xm, st.xp, st.ym, st.yp, st.zm, st.zp],
                      method=c["method"], seed=c["seed"], tol=c["tol"], restart=c["restart"], k=c["k"],
                      eb_rel=c["eb"], failures=c["failures"], baseline=base, final=fin.iteration,
                      converged=bool(fin.converged), n_prime=fin.iteration - base, recovered_from=recs,
                      ratios=ratios, norms=norms, seconds=time.time() - t0)
    print(name, {k: v for k, v in gold[name].items() if k not in ("norms", "ratios")}, flush=True)
    json.dump(gold, open(OUT, "w"), indent=1)
print("wrote", OUT)
