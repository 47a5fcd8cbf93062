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


CG_GOLD = os.path.join(ROOT, "tests", "golden", "config_golden.json")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config3", "config4_1e-4", "config4_1e-6", "config4_64_1e-4", "config4_64_1e-6"])
def test_configs_3_4_against_reference(dev, name):
    """BASELINE.json configs 3 (CG 128^3, failures at 100 and 300, eb 1e-5) and 4
    (GMRES(30) convection-diffusion, failure at the end of cycle 5, eb 1e-4 / 1e-6;
    32^3 and 64^3 -- the reference takes hours at 256^3) end to end on the GPU with
    the multi-failure protocol of tests/golden/make_config_golden.py: baseline and
    N' within +-1 of the real reference, residual norms within 1e-12 relative for
    the first iterations, every lossy checkpoint's ratio within 1e-3."""
    import json
    from paper_1805_07384_b200 import harness, solvers
    from paper_1805_07384_b200.compressor import CompressorConfig
    g = json.load(open(CG_GOLD)).get(name)
    if g is None:
        pytest.skip(f"{name} not in config_golden.json")
    a = solvers.StencilMatrix(*g["grid"], *g["stencil"])
    m = solvers.jacobi_preconditioner(a)
    b = torch.from_numpy(np.random.default_rng(g["seed"]).uniform(-1, 1, a.n_rows)).to(dev)
    cfg = solvers.SolveConfig(tolerance=g["tol"], restart_len=g["restart"], ckpt_intvl=g["k"],
                              max_iterations=100_000)
    s = solvers.init(g["method"], a, m, b, cfg)
    norms = [s.residual_norm]
    for _ in range(len(g["norms"]) - 1):
        s.step()
        norms.append(s.residual_norm)
    np.testing.assert_allclose(norms[:13], g["norms"][:13], rtol=1e-12)
    np.testing.assert_allclose(norms, g["norms"], rtol=1e-9)
    # block_version=1: the reference's block format, whose ratios the golden file holds
    res = harness.multi_failure_trial(g["method"], a, m, b, cfg, CompressorConfig.value_range_relative(g["eb_rel"]),
                                      g["failures"], g["k"], block_version=1)
    assert abs(res.baseline_n - g["baseline"]) <= 1, (res.baseline_n, g["baseline"])
    assert res.converged and list(res.recovered_from) == g["recovered_from"]
    assert abs(res.n_prime - g["n_prime"]) <= 1, (res.n_prime, g["n_prime"])
    np.testing.assert_allclose(res.ratios[:2], g["ratios"][:2], rtol=1e-3)
    # the checkpoint layer's default images (v3 blocks) reconstruct the same vectors:
    # same recoveries and iteration counts, ratios lower by the 24 B per 1024 symbols
    v3 = harness.multi_failure_trial(g["method"], a, m, b, cfg, CompressorConfig.value_range_relative(g["eb_rel"]),
                                     g["failures"], g["k"], baseline_n=res.baseline_n)
    assert v3.final_n == res.final_n and v3.recovered_from == res.recovered_from
    assert all(r3 < r1 for r3, r1 in zip(v3.ratios, res.ratios))


class _ThreadComm:
    """In-process stand-in for SlabComm (TEST ONLY): virtual ranks are host threads
    on one GPU, each on its own CUDA stream; halo planes and partial arrays move
    by device copies between the threads' buffers after a stream sync and a
    barrier.  No kernel ever waits for another rank's kernel."""

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def _publish(self, item):
        self.sh["items"][self.rank] = item
        torch.cuda.current_stream().synchronize()
        self.sh["barrier"].wait()

    def _done(self):
        torch.cuda.current_stream().synchronize()
        self.sh["barrier"].wait()

    def halo(self, buf, n, plane):
        self._publish((buf, n))
        if self.rank > 0:
            nb, nn = self.sh["items"][self.rank - 1]
            buf[0:plane].copy_(nb[nn:nn + plane])
        if self.rank < self.world - 1:
            nb, nn = self.sh["items"][self.rank + 1]
            buf[n + plane:n + 2 * plane].copy_(nb[plane:2 * plane])
        self._done()

    def allgather(self, out, local):
        self._publish(local)
        k = local.numel()
        for r in range(self.world):
            out[r * k:(r + 1) * k].copy_(self.sh["items"][r])
        self._done()
        return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_cg_bit_identical_on_device(dev, world):
    """The sharded CG kernels (slab offsets, halo planes, chunk partials) on the
    GPU: `world` virtual ranks give bit-identical norms and iterates to one GPU."""
    import threading
    from paper_1805_07384_b200 import solvers
    a = solvers.generate_laplacian3d(64)
    m = solvers.jacobi_preconditioner(a)
    cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=20)
    b = np.random.default_rng(4).uniform(-1, 1, a.n_rows)
    one = solvers.init("cg", a, m, torch.from_numpy(b).to(dev), cfg)
    ref_norms = [one.residual_norm]
    for _ in range(3):
        one.advance(17)
        ref_norms.append(one.residual_norm)
    shared = {"items": [None] * world, "barrier": threading.Barrier(world, timeout=120)}
    out = [None] * world
    errs = []

    def run(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                s = solvers.init("cg", a, m, torch.from_numpy(b).to(dev), cfg, comm=_ThreadComm(r, world, shared))
                norms = [s.residual_norm]
                for _ in range(3):
                    s.advance(17)
                    norms.append(s.residual_norm)
                out[r] = (norms, s.x.cpu().numpy(), s.iteration)
        except BaseException as exc:                    # a failed rank must not leave the others waiting
            errs.append(exc)
            shared["barrier"].abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    if errs:
        raise errs[0]
    for norms, _, it in out:
        assert norms == ref_norms and it == one.iteration
    xs = np.concatenate([o[1] for o in out])
    assert np.array_equal(xs.view(np.int64), one.x.cpu().numpy().view(np.int64))


@pytest.mark.gpu
def test_checkpoint_uses_producer_range(dev):
    """compress(x, value_range=solver.x_range) skips the value-range pass and gives
    the same block as the plain call (compressor.py:384-387 fused into the CG
    update kernel); the checkpoint layer passes the record automatically."""
    from paper_1805_07384_b200 import _native, checkpoint as ckpt, compressor, solvers
    a = solvers.generate_laplacian3d(48)
    s = solvers.init("cg", a, solvers.jacobi_preconditioner(a),
                     torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, a.n_rows)).to(dev),
                     solvers.SolveConfig(tolerance=1e-8, restart_len=20))
    s.advance(23)
    for eb in (1e-3, 1e-5):
        cfg = compressor.CompressorConfig.value_range_relative(eb)
        plain = compressor.compress(s.x, cfg).to_bytes()
        ctx = _native.context(0)
        n0 = ctx.lib.lc_launch_count(ctx.h)
        ranged = compressor.compress(s.x, cfg, value_range=s.x_range).to_bytes()
        n1 = ctx.lib.lc_launch_count(ctx.h)
        assert ranged == plain
        img, _ = ckpt.checkpoint_lossy(s, cfg, ckpt.StorageTarget(), block_version=1)
        assert img.payload == plain
        assert n1 - n0 >= 1


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_config4_full_size_state_compresses_exactly(dev):
    """BASELINE.json config 4 at its full size: the GMRES(30) iterate of the 256^3
    convection-diffusion problem after 120 iterations, eb_rel 1e-6 (all 65,536 symbols in
    use, ~760k escapes, periodic offset maps in the warp scans, ~19 chunk-prediction
    resumes).  This vector once left a lane split off from its warp inside the map scan
    (endless tile loop in pass A, garbage codes): blocks must equal the oracle's byte for
    byte with and without the producer's range, and v1 / v3 must reconstruct bit for bit."""
    from paper_1805_07384_b200 import compressor, solvers
    from oracle import oracle as orc
    a = solvers.generate_convdiff3d(256)
    m = solvers.jacobi_preconditioner(a)
    b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, a.n_rows)).to(dev)
    cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=30, ckpt_intvl=60, max_iterations=100_000)
    s = solvers.init("gmres", a, m, b, cfg)
    s.advance(120)
    x = s.x.detach().clone()
    ref = orc.compress(x.cpu().numpy(), "value_range_relative", 1e-6)
    want = orc.to_bytes(ref)
    cc = compressor.CompressorConfig.value_range_relative(1e-6)
    assert compressor.compress(x, cc, block_version=1).to_bytes() == want
    assert compressor.compress(x, cc, block_version=1, value_range=s.x_range).to_bytes() == want
    for version in (1, 3):
        rec = compressor.decompress(compressor.compress(x, cc, block_version=version))
        assert np.array_equal(rec.view(np.int64), ref["recon"].view(np.int64)), version
