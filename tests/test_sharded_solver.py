"""Slab-sharded solvers (BASELINE.json config 5) at world size 2
over gloo on CPU: the host logic of paper_1805_07384_b200.solvers with comm
(halo exchange of boundary planes, all-gather of the per-chunk reduction
partials, batched iterations, CG restarts, GMRES cycles) driven through the
CPU double of the device kernels (tests/numpy_ops.py).  Sharded runs must be
BIT-identical to the one-process run: same residual norms, same iterates,
same iteration counts."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_1805_07384_b200 import solvers as S  # noqa: E402
from numpy_ops import NumpyOps  # noqa: E402

GRID = (64, 64, 8)                    # nx*ny = 4096: one reduction chunk per plane
CASES = {
    "cg": (S.StencilMatrix(*GRID, 6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0),
           S.SolveConfig(tolerance=1e-8, restart_len=7, ckpt_intvl=7), 45),
    "jacobi": (S.StencilMatrix(*GRID, 6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0),
               S.SolveConfig(tolerance=1e-6), 30),
    "gmres": (S.StencilMatrix(*GRID, 6.175, -1.1, -1.0, -1.05, -1.0, -1.025, -1.0),
              S.SolveConfig(tolerance=1e-8, restart_len=6), 20),
}


def _b():
    return np.random.default_rng(11).uniform(-1, 1, int(np.prod(GRID)))


def _run(method, comm):
    a, cfg, steps = CASES[method]
    m = S.jacobi_preconditioner(a)
    s = S.init(method, a, m, _b(), cfg, comm=comm, ops=NumpyOps())
    norms = [s.residual_norm]
    for _ in range(steps // 3):                         # step() one at a time
        s.step()
        norms.append(s.residual_norm)
    s.advance(steps - steps // 3)                        # then one batch
    norms.append(s.residual_norm)
    return np.array(norms), s.x.numpy().copy(), s.iteration


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        comm = S.SlabComm()
        for method in CASES:
            norms, x, it = _run(method, comm)
            np.savez(os.path.join(outdir, f"{method}_{rank}.npz"), norms=norms, x=x, it=it)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded(tmp_path_factory):
    out = tmp_path_factory.mktemp("shard")
    mp.start_processes(_worker, args=(_free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    return out


@pytest.mark.parametrize("method", list(CASES))
def test_world2_bit_identical_to_one_process(sharded, method):
    norms1, x1, it1 = _run(method, None)
    r0 = np.load(os.path.join(sharded, f"{method}_0.npz"))
    r1 = np.load(os.path.join(sharded, f"{method}_1.npz"))
    assert int(r0["it"]) == int(r1["it"]) == it1
    for r in (r0, r1):
        assert np.array_equal(r["norms"].view(np.int64), norms1.view(np.int64)), method
    xs = np.concatenate([r0["x"], r1["x"]])
    assert np.array_equal(xs.view(np.int64), x1.view(np.int64)), method


def test_batched_equals_stepwise():
    """advance(k) (one host round trip, device status gating) == k single steps."""
    a, cfg, _ = CASES["cg"]
    m = S.jacobi_preconditioner(a)
    s1 = S.init("cg", a, m, _b(), cfg, ops=NumpyOps())
    for _ in range(25):
        s1.step()
    s2 = S.init("cg", a, m, _b(), cfg, ops=NumpyOps())
    assert s2.advance(25) == 25
    assert np.array_equal(s1.x.numpy(), s2.x.numpy()) and s1.residual_norm == s2.residual_norm


def test_batch_stops_at_convergence():
    """Iterations queued past convergence do nothing: the iteration count and x
    are those of the step that converged (solvers.py:271-276)."""
    a = S.StencilMatrix(16, 16, 1, 4.0, -1.0, -1.0, -1.0, -1.0)
    cfg = S.SolveConfig(tolerance=1e-6, restart_len=1000)
    m = S.jacobi_preconditioner(a)
    b = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    s1 = S.init("cg", a, m, b, cfg, ops=NumpyOps())
    while not s1.converged:
        s1.step()
    s2 = S.init("cg", a, m, b, cfg, ops=NumpyOps())
    s2.advance(s1.iteration + 40)
    assert s2.converged and s2.iteration == s1.iteration
    assert np.array_equal(s1.x.numpy(), s2.x.numpy())
    with pytest.raises(S.ParameterError):
        s2.step()


def test_x_range_record():
    """The update kernel's range record equals the iterate's min/max (checkpoints
    skip the compressor's range pass with it)."""
    a, cfg, _ = CASES["cg"]
    s = S.init("cg", a, S.jacobi_preconditioner(a), _b(), cfg, ops=NumpyOps())
    assert s.x_range is None                            # x from outside: no record
    s.advance(5)
    rr = s.x_range.numpy()
    x = s.x.numpy()
    assert rr[0] == x.min() and rr[1] == x.max() and rr[3] == 0.0 and rr[2] == np.max(np.abs(np.diff(x)))


def test_uneven_split_rejected():
    class Comm:
        rank, world = 0, 3
    a, cfg, _ = CASES["cg"]
    with pytest.raises(S.ParameterError, match="split evenly"):
        S.init("cg", a, S.jacobi_preconditioner(a), _b(), cfg, comm=Comm(), ops=NumpyOps())


@pytest.mark.parametrize("name", ["jac2d", "cg3d", "gmres3d"])
def test_host_logic_matches_reference_norms(name):
    """The solver host logic (restarts, GMRES cycles, Givens, batching) over the
    CPU double reproduces the REAL reference's residual norms
    (tests/golden/solver_golden.npz) within 1e-12 relative."""
    sg = np.load(os.path.join(HERE, "golden", "solver_golden.npz"))
    st = sg[name + "/stencil"]
    a = S.StencilMatrix(int(st[0]), int(st[1]), int(st[2]), *[float(v) for v in st[3:]])
    tol, maxit, rl, ck, _ = sg[name + "/cfg"]
    cfg = S.SolveConfig(tolerance=float(tol), max_iterations=int(maxit), restart_len=int(rl), ckpt_intvl=int(ck))
    method = ["jacobi", "cg", "gmres"][int(sg[name + "/method"][0])]
    s = S.init(method, a, S.jacobi_preconditioner(a), sg[name + "/b"], cfg, ops=NumpyOps())
    norms = [s.residual_norm]
    for _ in range(len(sg[name + "/norms"]) - 1):
        s.step()
        norms.append(s.residual_norm)
    np.testing.assert_allclose(norms, sg[name + "/norms"], rtol=1e-12)
    base = S.solve_to_convergence(S.init(method, a, S.jacobi_preconditioner(a), sg[name + "/b"], cfg,
                                         ops=NumpyOps()))
    assert abs(base.iteration - int(sg[name + "/baseline"][0])) <= 1
