"""GPU solver harness against the real reference (tests/golden/make_solver_golden.py).

Bars (BASELINE.json north star): stencil SpMV and Jacobi iterates bit-exact
with the reference's CSR spmv / numpy updates; residual norms within 1e-12
relative (parallel vs numpy/BLAS summation order); baseline iteration counts
and extra iterations after restart (N') within +-1 of the reference.
Config 1 (poisson2d(256), Jacobi, k=10, failure at 200) runs when its golden
entry is present (reference: baseline 112,797, N' = -61)."""

import os

import numpy as np
import pytest

from tests.conftest import ROOT

SG = os.path.join(ROOT, "tests", "golden", "solver_golden.npz")
METHODS = ["jacobi", "cg", "gmres"]
NORM_RTOL = 1e-12


@pytest.fixture(scope="module")
def sg():
    return np.load(SG, allow_pickle=False)


def _names(z):
    return sorted({k.split("/")[0] for k in z.files})


def _case(sg, name):
    from paper_1805_07384_b200 import solvers
    st = sg[name + "/stencil"]
    a = solvers.StencilMatrix(int(st[0]), int(st[1]), int(st[2]), *[float(v) for v in st[3:]])
    tol, maxit, rl, ck, eb = sg[name + "/cfg"]
    cfg = solvers.SolveConfig(tolerance=float(tol), max_iterations=int(maxit), restart_len=int(rl),
                              ckpt_intvl=int(ck))
    return a, cfg, float(eb), METHODS[int(sg[name + "/method"][0])]


def _csr_spmv(a, x):
    """The reference's sequential CSR accumulation (sparse.py:21-28), vectorised over rows."""
    ro, ci, va = a.to_csr_arrays()
    counts = np.diff(ro)
    acc = np.zeros(a.n_rows)
    for t in range(counts.max()):
        rows = np.nonzero(counts > t)[0]
        idx = ro[rows] + t
        acc[rows] = acc[rows] + va[idx] * x[ci[idx]]
    return acc


def test_csr_layout_matches_reference_generator():
    """StencilMatrix's CSR equals generate_poisson2d's (sparse.py:184-206) entry order."""
    from paper_1805_07384_b200.solvers import StencilMatrix
    m = 5
    a = StencilMatrix(m, m, 1, 4.0, -1.0, -1.0, -1.0, -1.0)
    ro, ci, va = a.to_csr_arrays()
    rows, cols, vals = [], [], []
    for i in range(m):
        for j in range(m):
            k = i * m + j
            if i > 0:
                rows.append(k), cols.append(k - m), vals.append(-1.0)
            if j > 0:
                rows.append(k), cols.append(k - 1), vals.append(-1.0)
            rows.append(k), cols.append(k), vals.append(4.0)
            if j < m - 1:
                rows.append(k), cols.append(k + 1), vals.append(-1.0)
            if i < m - 1:
                rows.append(k), cols.append(k + m), vals.append(-1.0)
    assert np.array_equal(ci, cols) and np.array_equal(va, vals)
    assert np.array_equal(np.repeat(np.arange(m * m), np.diff(ro)), rows)


torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


@pytest.mark.gpu
def test_spmv_bit_exact(dev):
    from paper_1805_07384_b200 import solvers
    rng = np.random.default_rng(5)
    for a in (solvers.StencilMatrix(33, 17, 1, 4.0, -1.0, -1.0, -1.0, -1.0), solvers.generate_laplacian3d(9),
              solvers.generate_convdiff3d(7)):
        x = rng.normal(size=a.n_rows)
        y = solvers.spmv(a, torch.from_numpy(x).to(dev)).cpu().numpy()
        assert np.array_equal(y.view(np.int64), _csr_spmv(a, x).view(np.int64))


@pytest.mark.gpu
def test_jacobi_iterates_and_norms(dev, sg):
    from paper_1805_07384_b200 import solvers
    a, cfg, _, method = _case(sg, "jac2d")
    m = solvers.jacobi_preconditioner(a)
    s = solvers.init(method, a, m, torch.from_numpy(sg["jac2d/b"]).to(dev), cfg)
    for _ in range(int(sg["jac2d/n_steps"][0])):
        s.step()
    assert np.array_equal(s.x.cpu().numpy().view(np.int64), sg["jac2d/x_steps"].view(np.int64))


@pytest.mark.gpu
def test_residual_norms_all_methods(dev, sg):
    from paper_1805_07384_b200 import solvers
    for name in ("jac2d", "cg3d", "gmres3d"):
        a, cfg, _, method = _case(sg, name)
        m = solvers.jacobi_preconditioner(a)
        s = solvers.init(method, a, m, torch.from_numpy(sg[name + "/b"]).to(dev), cfg)
        norms = [s.residual_norm]
        for _ in range(len(sg[name + "/norms"]) - 1):
            s.step()
            norms.append(s.residual_norm)
        np.testing.assert_allclose(norms, sg[name + "/norms"], rtol=NORM_RTOL, err_msg=name)


@pytest.mark.gpu
def test_n_prime_matches_reference(dev, sg):
    from paper_1805_07384_b200 import harness, solvers
    from paper_1805_07384_b200.compressor import CompressorConfig
    for name in _names(sg):
        if name == "config1":
            continue
        a, cfg, eb, method = _case(sg, name)
        m = solvers.jacobi_preconditioner(a)
        res = harness.measure_n_prime(method, a, m, torch.from_numpy(sg[name + "/b"]).to(dev), cfg,
                                      CompressorConfig.value_range_relative(eb), sg[name + "/inject"])
        assert abs(res.baseline_n - int(sg[name + "/baseline"][0])) <= 1, name
        np.testing.assert_allclose(res.values(), sg[name + "/nprime"], atol=1, err_msg=name)


@pytest.mark.gpu
def test_config1_n_prime(dev, sg):
    """BASELINE.json config 1 end to end on the GPU: N' within +-1 of the reference."""
    if "config1/baseline" not in sg.files:
        pytest.skip("config-1 golden not generated (make_solver_golden.py --full)")
    from paper_1805_07384_b200 import harness, solvers
    from paper_1805_07384_b200.compressor import CompressorConfig
    a, cfg, eb, method = _case(sg, "config1")
    m = solvers.jacobi_preconditioner(a)
    res = harness.measure_n_prime(method, a, m, torch.from_numpy(sg["config1/b"]).to(dev), cfg,
                                  CompressorConfig.value_range_relative(eb), sg["config1/inject"])
    assert abs(res.baseline_n - int(sg["config1/baseline"][0])) <= 1
    np.testing.assert_allclose(res.values(), sg["config1/nprime"], atol=1)


TG = os.path.join(ROOT, "tests", "golden", "trial_golden.json")


@pytest.mark.gpu
def test_run_trial_matches_reference(dev, reference):
    """The reference's own Poisson-failure event loop (simulate.run_trial) driving the
    GPU workload, against the same loop over its CPU workload (golden reports): identical
    event bookkeeping for Jacobi (bit-identical iterates); CG/GMRES recoveries may shift
    the convergence step by one per recovery."""
    import json
    from lossyckpt import simulate
    from lossyckpt.compressor import CompressorConfig as RefConfig
    from paper_1805_07384_b200 import harness
    for case in json.load(open(TG)):
        c = dict(case["config"])
        eb = c.pop("eb_rel")
        seed = c["seed"]
        if eb is not None:
            c["compressor_config"] = RefConfig.value_range_relative(eb)
        cfg = simulate.SimConfig(**c)
        rep = simulate.run_trial(cfg, seed, workload=harness.GpuSolverWorkload(cfg))
        ref = case["report"]
        assert rep.converged == ref["converged"] and rep.diverged == ref["diverged"], c
        if c["method"] == "jacobi":
            for k, v in ref.items():
                if isinstance(v, float):
                    assert abs(getattr(rep, k) - v) <= 1e-9 * max(1.0, abs(v)), (k, c)
                else:
                    assert getattr(rep, k) == v, (k, c)
        else:
            assert abs(rep.iterations_final - ref["iterations_final"]) <= 1 + ref["n_recoveries"], c
