"""On-GPU solver harness (north star "Solver harness").

Mirrors lossyckpt/solvers.py (SolveConfig, JacobiSolver, CgSolver,
GmresSolver, init, rebuild_from_solution, solve_to_convergence; solvers.py:
23-276) for the constant-coefficient stencil matrices of BASELINE.json's
configs, with state vectors as torch CUDA float64 tensors and every vector
operation in the hand-written kernels of csrc/lc_krylov.cu through the C ABI.

* Scalars stay on the device (lc_kscalars): CG/Jacobi queue many iterations
  per host round trip (`advance`, `solve_to_convergence`); kernels queued
  after convergence do nothing.  GMRES reads one column of H per iteration
  (its Givens rotations are host scalars, as in the reference).
* Slab sharding (config 5): with `comm` (SlabComm over torch.distributed,
  NCCL on the GPU) each rank owns nz/world z-planes; the stencil's halo
  planes move by batched send/recv and the dot products all-gather per-chunk
  partials that every rank folds in the same fixed order, so a sharded run
  is bit-identical to the one-GPU run.
* The kernel that produces x also emits its value range (`x_range`), so a
  lossy checkpoint skips the compressor's range pass.

Arithmetic follows the reference operation by operation: y = A x is
accumulated in CSR column order with unfused multiply/add (bit-identical to
sparse.py:21-28), updates are one rounded multiply and one rounded add as in
the numpy expressions, so Jacobi iterates are bit-identical to the
reference.  Dot products and norms use a fixed-order chunked reduction
instead of numpy/BLAS's order, so the step at which ||r|| <= tol*||b|| first
holds can differ by one iteration (the north star's +-1 tolerance).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from .errors import BreakdownError, DimensionMismatchError, ParameterError


@dataclass(frozen=True)
class SolveConfig:
    """Iteration control shared by all methods (solvers.py:23-41)."""

    tolerance: float = 1e-8
    max_iterations: int = 100_000
    restart_len: int = 30
    ckpt_intvl: int = 30

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ParameterError("tolerance must be positive")
        if self.max_iterations < 1 or self.restart_len < 1 or self.ckpt_intvl < 1:
            raise ParameterError("max_iterations, restart_len, ckpt_intvl must be >= 1")


class LcStencil(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("c", ctypes.c_double), ("xm", ctypes.c_double), ("xp", ctypes.c_double),
                ("ym", ctypes.c_double), ("yp", ctypes.c_double), ("zm", ctypes.c_double),
                ("zp", ctypes.c_double)]


@dataclass(frozen=True)
class StencilMatrix:
    """Constant-coefficient 7-point stencil on nx*ny*nz points (x fastest),
    Dirichlet boundary (missing neighbours dropped).  Plays the role of
    SparseMatrixCsr for the configs' matrices; `to_csr_arrays` gives the
    equivalent CSR (column-sorted rows) for checks."""

    nx: int
    ny: int
    nz: int
    c: float
    xm: float = 0.0
    xp: float = 0.0
    ym: float = 0.0
    yp: float = 0.0
    zm: float = 0.0
    zp: float = 0.0

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ParameterError("grid sides must be >= 1")

    @property
    def n_rows(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_cols(self) -> int:
        return self.n_rows

    def abi(self) -> LcStencil:
        return LcStencil(self.nx, self.ny, self.nz, self.c, self.xm, self.xp, self.ym, self.yp, self.zm, self.zp)

    def to_csr_arrays(self):
        """(row_offsets, col_indices, values) in the reference's CSR order."""
        nx, ny, nz = self.nx, self.ny, self.nz
        k = np.arange(self.n_rows)
        iz, rem = np.divmod(k, nx * ny)
        iy, ix = np.divmod(rem, nx)
        terms = [(iz > 0, -nx * ny, self.zm), (iy > 0, -nx, self.ym), (ix > 0, -1, self.xm),
                 (np.ones_like(k, bool), 0, self.c), (ix < nx - 1, 1, self.xp),
                 (iy < ny - 1, nx, self.yp), (iz < nz - 1, nx * ny, self.zp)]
        present = np.stack([t[0] & (t[2] != 0.0) | (t[1] == 0) for t in terms], axis=1)
        cols = np.stack([k + t[1] for t in terms], axis=1)
        vals = np.stack([np.full(k.shape, t[2]) for t in terms], axis=1)
        counts = present.sum(axis=1)
        ro = np.concatenate([[0], np.cumsum(counts)])
        return ro, cols[present], vals[present]


def generate_poisson2d(m: int, device="cuda"):
    """5-point Laplacian on an m x m grid (diagonal 4, neighbours -1) and b = ones
    (sparse.py:184-206; row-major k = i*m + j: x is j, y is i)."""
    import torch
    if m < 2:
        raise ParameterError("grid side length must be >= 2")
    a = StencilMatrix(m, m, 1, 4.0, -1.0, -1.0, -1.0, -1.0, 0.0, 0.0)
    return a, torch.ones(m * m, dtype=torch.float64, device=device)


def generate_laplacian3d(m: int) -> StencilMatrix:
    """7-point Laplacian on an m^3 grid (diagonal 6, neighbours -1), Dirichlet
    (BASELINE.json configs 3 and 5)."""
    if m < 2:
        raise ParameterError("grid side length must be >= 2")
    return StencilMatrix(m, m, m, 6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0)


def generate_convdiff3d(m: int, velocity=(1.0, 0.5, 0.25), scale: float = 0.1) -> StencilMatrix:
    """Diffusion 1 plus first-order upwind convection with constant velocity
    velocity * scale / h on an m^3 grid, scaled by h^2 (BASELINE.json config 4;
    the generator is harness-defined there).  For a velocity component v >= 0 the
    upwind term v*h*(u_i - u_{i-1}) adds v*h to the centre and -v*h to the
    lower neighbour."""
    if m < 2:
        raise ParameterError("grid side length must be >= 2")
    vx, vy, vz = (scale * v for v in velocity)
    if min(vx, vy, vz) < 0:
        raise ParameterError("upwind generator expects non-negative velocity components")
    return StencilMatrix(m, m, m, 6.0 + vx + vy + vz, -1.0 - vx, -1.0, -1.0 - vy, -1.0, -1.0 - vz, -1.0)


@dataclass(frozen=True)
class DiagonalPreconditioner:
    """Diagonal preconditioner stored as the (constant) inverse diagonal (sparse.py:128-147)."""

    inverse_diagonal: float
    n: int

    def __post_init__(self):
        if not math.isfinite(self.inverse_diagonal) or self.inverse_diagonal == 0.0:
            raise ParameterError("inverse diagonal entries must be finite and nonzero")


def jacobi_preconditioner(a: StencilMatrix) -> DiagonalPreconditioner:
    """M = diag(A) (sparse.py:160-167)."""
    if a.c == 0.0:
        raise ParameterError("zero diagonal")
    return DiagonalPreconditioner(1.0 / a.c, a.n_rows)


# --- device primitives -----------------------------------------------------------

def _ctx(t):
    return _native.context(t.device.index or 0)


def _check(ctx, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc}): {ctx.error()}")


def spmv(a: StencilMatrix, x):
    """y = A @ x on the device (sparse.py:150-157)."""
    import torch
    if x.numel() != a.n_cols:
        raise DimensionMismatchError(f"matrix has {a.n_cols} columns, vector has {x.numel()} entries")
    x = x.contiguous()
    y = torch.empty_like(x)
    ctx = _ctx(x)
    st = a.abi()
    _check(ctx, ctx.lib.lc_stencil_apply_f64(ctx.h, ctypes.addressof(st), x.data_ptr(), y.data_ptr()), "spmv")
    return y


def dot(a, b) -> float:
    ctx = _ctx(a)
    out = ctypes.c_double()
    _check(ctx, ctx.lib.lc_dot_f64(ctx.h, a.data_ptr(), b.data_ptr(), a.numel(), None, ctypes.byref(out)), "dot")
    return out.value


def axpy(alpha: float, x, y):
    """y += alpha * x (one rounded multiply, one rounded add)."""
    ctx = _ctx(x)
    _check(ctx, ctx.lib.lc_axpy_f64(ctx.h, float(alpha), None, 1.0, x.data_ptr(), y.data_ptr(), x.numel()), "axpy")


# --- device-resident solvers (csrc/lc_krylov.cu) ---------------------------------

CHUNK = 4096                      # LC_KR_CHUNK_ELEMS: elements per reduction partial
KS_RUNNING, KS_CONVERGED, KS_BREAKDOWN, KS_NONFINITE = 0, 1, 2, 3
(KOP_DOT, KOP_NORM, KOP_ALPHA, KOP_BETA, KOP_REBUILD_INIT, KOP_REBUILD_STEP, KOP_RESID,
 KOP_RESID_INIT) = range(8)
BATCH = 256                       # steps queued per host sync in advance()/solve_to_convergence


class LcSlab(ctypes.Structure):
    _fields_ = [("st", LcStencil), ("z0", ctypes.c_int64), ("nzl", ctypes.c_int64)]


class LcKScalars(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("pq", ctypes.c_double), ("alpha", ctypes.c_double),
                ("beta", ctypes.c_double), ("rr", ctypes.c_double), ("res", ctypes.c_double),
                ("tol_abs", ctypes.c_double), ("spare", ctypes.c_double), ("iteration", ctypes.c_int64),
                ("status", ctypes.c_int32), ("pad", ctypes.c_int32)]


assert ctypes.sizeof(LcKScalars) == 80


def _p(t, off=0):
    """Device address of element `off` of tensor t (None passes through)."""
    return None if t is None else t.data_ptr() + 8 * off


class DeviceOps:
    """The solvers' vector operations: the hand-written kernels of
    csrc/lc_krylov.cu through the C ABI (the only product implementation;
    a solver step never calls torch arithmetic).  Vectors are torch float64
    CUDA tensors; `scalars()` is an lc_kscalars block in HBM."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ParameterError("DeviceOps needs a CUDA device")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        # the solver's kernels are ordered on the stream current at construction
        # (the calling thread's codec context for that stream)
        self.stream = torch.cuda.current_stream(self.device.index).cuda_stream
        self.lib = _native.library()

    def _call(self, name, *args):
        ctx = _native.bind_stream(self.device.index, self.stream)
        rc = getattr(self.lib, name)(ctx.h, *args)
        if rc != 0:
            _check(ctx, rc, name)

    # storage
    def empty(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device=self.device)

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def as_vector(self, v):
        t = self.torch.as_tensor(v, dtype=self.torch.float64)
        return t.to(self.device).reshape(-1).contiguous()

    def scalars(self):
        return self.torch.zeros(10, dtype=self.torch.float64, device=self.device)

    def range_record(self):
        return self.torch.zeros(4, dtype=self.torch.float64, device=self.device)

    def set_scalars(self, sc, **fields):
        s = LcKScalars()
        for k, v in fields.items():
            setattr(s, k, v)
        host = self.torch.frombuffer(bytearray(bytes(s)), dtype=self.torch.float64)
        sc.copy_(host)

    def get_scalars(self, sc) -> LcKScalars:
        host = sc.cpu().numpy().tobytes()                # waits for the stream
        return LcKScalars.from_buffer_copy(host)

    def read(self, t):
        return t.cpu().numpy()

    def write(self, dst, host_values):
        dst.copy_(self.torch.as_tensor(np.asarray(host_values, dtype=np.float64)))

    # kernels (pointers: vh = first local element of a halo vector)
    def spmv(self, slab, vh, off, y, part, sc):
        self._call("lc_kr_spmv_f64", ctypes.byref(slab), _p(vh, off), _p(y), _p(part), _p(sc))

    def residual(self, slab, xh, off, b, r, inv, z, zoff, part, sc_gate):
        self._call("lc_kr_residual_f64", ctypes.byref(slab), _p(xh, off), _p(b), _p(r), float(inv), _p(z, zoff),
                   _p(part), _p(sc_gate))

    def cg_update(self, n, p, poff, q, x, xoff, r, inv, sc, part, rparts):
        self._call("lc_kr_cg_update_f64", n, _p(p, poff), _p(q), _p(x, xoff), _p(r), float(inv), _p(sc), _p(part),
                   _p(rparts))

    def cg_dir(self, n, r, p, poff, inv, sc):
        self._call("lc_kr_cg_dir_f64", n, _p(r), _p(p, poff), float(inv), _p(sc))

    def jacobi(self, slab, inv, xh, xoff, rh, roff, b, x2, x2off, r2, r2off, sc, part, rparts):
        self._call("lc_kr_jacobi_f64", ctypes.byref(slab), float(inv), _p(xh, xoff), _p(rh, roff), _p(b),
                   _p(x2, x2off), _p(r2, r2off), _p(sc), _p(part), _p(rparts))

    def dot(self, n, a, aoff, b, boff, part, sc):
        self._call("lc_kr_dot_f64", n, _p(a, aoff), _p(b, boff), _p(part), _p(sc))

    def subh(self, n, x, xoff, y, h, hoff, sc):
        self._call("lc_kr_subh_f64", n, _p(x, xoff), _p(y), _p(h, hoff), _p(sc))

    def div(self, n, x, y, yoff, d, doff, sc):
        self._call("lc_kr_div_f64", n, _p(x), _p(y, yoff), _p(d, doff), _p(sc))

    def combine(self, n, j, basis, boff, ld, yv, xbase, x, xoff, rparts):
        self._call("lc_kr_combine_f64", n, int(j), _p(basis, boff), ld, _p(yv), _p(xbase, boff), _p(x, xoff),
                   _p(rparts))

    def fold(self, part, width, nch, op, sc, out=None, outoff=0, rparts=None, nrp=0, rout=None):
        self._call("lc_kr_fold_f64", _p(part), int(width), nch, int(op), _p(sc), _p(out, outoff), _p(rparts), nrp,
                   _p(rout))


class SlabComm:
    """torch.distributed plumbing of a z-slab-sharded solver:
    halo exchange of the boundary planes with the neighbouring ranks
    (batched send/recv) and the all-gather of per-chunk reduction partials
    (the dot-product "allreduce": every rank folds the same global array in
    the same order, so results do not depend on the number of ranks).  NCCL
    over NVLink for CUDA tensors, gloo for CPU tensors."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def halo(self, buf, n, plane):
        """buf = [lower halo | n local | upper halo], halo planes of `plane` elements."""
        if self.world == 1:
            return
        d = self.dist
        ops = []
        peer = lambda r: d.get_global_rank(self.group, r) if self.group is not None else r  # noqa: E731
        if self.rank > 0:
            ops.append(d.P2POp(d.isend, buf[plane:2 * plane], peer(self.rank - 1), self.group))
            ops.append(d.P2POp(d.irecv, buf[0:plane], peer(self.rank - 1), self.group))
        if self.rank < self.world - 1:
            ops.append(d.P2POp(d.isend, buf[n:n + plane], peer(self.rank + 1), self.group))
            ops.append(d.P2POp(d.irecv, buf[n + plane:n + 2 * plane], peer(self.rank + 1), self.group))
        for w in d.batch_isend_irecv(ops):
            w.wait()

    def allgather(self, out, local):
        if self.world == 1:
            return local
        self.dist.all_gather_into_tensor(out, local, group=self.group)
        return out


class _Layout:
    """Slab of the global stencil owned by this rank (z-planes split evenly)."""

    def __init__(self, a: StencilMatrix, comm):
        world = comm.world if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        if a.nz % world:
            raise ParameterError(f"nz = {a.nz} planes do not split evenly over {world} ranks")
        self.plane = a.nx * a.ny
        if world > 1 and self.plane % CHUNK:
            raise ParameterError(f"sharded solvers need nx*ny to be a multiple of {CHUNK} (reduction chunks)")
        self.world, self.rank = world, rank
        self.nzl = a.nz // world
        self.z0 = rank * self.nzl
        self.n = self.plane * self.nzl
        self.halo = self.plane if world > 1 else 0
        self.nch = -(-self.n // CHUNK)
        self.nch_global = self.nch * world
        self.slab = LcSlab(a.abi(), self.z0, self.nzl)


class _SolverBase:
    """State machine shared by the methods (solvers.py:44-89).  Vectors are
    slabs of the global problem when `comm` is given (CG and GMRES: NCCL halo
    exchange + partial all-gather; one GPU otherwise); `ops` is the vector
    backend (DeviceOps; tests may substitute a CPU double for the sharding
    logic)."""

    method = "?"

    def __init__(self, a: StencilMatrix, m: DiagonalPreconditioner, b, config: SolveConfig,
                 x=None, iteration: int = 0, comm=None, ops=None, device=None):
        if ops is None:
            import torch
            dev = device
            if dev is None:
                dev = b.device if (isinstance(b, torch.Tensor) and b.is_cuda) else "cuda"
            ops = DeviceOps(dev)
        self.ops = ops
        self.comm = comm
        L = self._lay = _Layout(a, comm)
        b = ops.as_vector(b)
        if b.numel() == a.n_rows and L.world > 1:
            b = b[L.z0 * L.plane:(L.z0 + L.nzl) * L.plane].contiguous()
        if b.numel() != L.n:
            raise DimensionMismatchError("matrix and right-hand side sizes differ")
        if m.n != a.n_rows:
            raise DimensionMismatchError("preconditioner size differs from matrix")
        if iteration < 0:
            raise ParameterError("iteration index must be non-negative")
        self.a, self.m, self.b = a, m, b
        self.config = config
        self.iteration = iteration
        self._planned = iteration
        self._xh = ops.zeros(L.n + 2 * L.halo)
        if x is not None:
            xv = ops.as_vector(x)
            if xv.numel() == a.n_rows and L.world > 1:
                xv = xv[L.z0 * L.plane:(L.z0 + L.nzl) * L.plane]
            if xv.numel() != L.n:
                raise DimensionMismatchError("initial guess size differs from matrix")
            self._xh[L.halo:L.halo + L.n].copy_(xv)
        self._part = ops.empty(2 * L.nch)
        self._gpart = ops.empty(2 * L.nch_global) if L.world > 1 else None
        self._rparts = ops.empty(6 * L.nch)          # per-chunk range records (LcKrRange, 48 B)
        self._range = ops.range_record()
        self._range_valid = False
        self._out = ops.zeros(4)
        self.sc = ops.scalars()
        self.norm_b = math.sqrt(self._global_dot(b, 0, b, 0))
        self._tol_abs = config.tolerance * self.norm_b
        ops.set_scalars(self.sc, tol_abs=self._tol_abs, iteration=iteration, status=KS_RUNNING)
        self.residual_norm = math.inf
        self.converged = False
        self._rebuild()

    # -- plumbing
    @property
    def x(self):
        """The iterate (this rank's slab), a view of the solver's buffer."""
        L = self._lay
        return self._xh[L.halo:L.halo + L.n]

    @property
    def x_range(self):
        """Device range record (vmin, vmax, maxstep, nonfinite) of x computed by
        the kernel that produced it, or None (lossy checkpoints skip the
        value-range pass with it: compressor.compress(value_range=...))."""
        return self._range if self._range_valid else None

    def _halo(self, buf):
        if self.comm is not None:
            self.comm.halo(buf, self._lay.n, self._lay.plane)

    def _gathered(self, width):
        L = self._lay
        local = self._part[:width * L.nch]
        if self.comm is None or L.world == 1:
            return local
        return self.comm.allgather(self._gpart[:width * L.nch_global], local)

    def _global_dot(self, a, aoff, b, boff) -> float:
        L = self._lay
        self.ops.dot(L.n, a, aoff, b, boff, self._part, None)
        self.ops.fold(self._gathered(1), 1, L.nch_global, KOP_DOT, None, out=self._out)
        return float(self.ops.read(self._out)[0])

    def _sync(self):
        """Read the device scalars (one host round trip) and raise on a breakdown."""
        s = self.ops.get_scalars(self.sc)
        self.iteration = int(s.iteration)
        self._planned = self.iteration
        self.residual_norm = float(s.res)
        self.converged = s.status == KS_CONVERGED
        if s.status == KS_BREAKDOWN:
            raise BreakdownError("CG breakdown: zero curvature or zero rho", self.iteration)
        if s.status == KS_NONFINITE:
            raise BreakdownError("residual norm is not finite", self.iteration)
        return s

    def _rebuild(self):
        raise NotImplementedError

    def _enqueue_step(self):
        raise NotImplementedError

    def _check_steppable(self):
        if self.converged:
            raise ParameterError("step() called on a converged solver")
        if self.iteration >= self.config.max_iterations:
            raise ParameterError("step() called at the iteration cap")

    def step(self):
        """One iteration (solvers.py step()); one host round trip."""
        self._check_steppable()
        self._enqueue_step()
        self._sync()
        return self

    def advance(self, k: int) -> int:
        """Up to k iterations, stopping at convergence or the cap, with one host
        round trip: every kernel of an iteration queued after the solver
        stopped returns at once (device status word).  Returns the iterations
        taken."""
        start = self.iteration
        k = min(int(k), self.config.max_iterations - self.iteration)
        if k <= 0 or self.converged:
            return 0
        for _ in range(k):
            self._enqueue_step()
        self._sync()
        return self.iteration - start


class JacobiSolver(_SolverBase):
    """x <- x + M^-1 (b - A x) (solvers.py:92-110); one fused kernel + one fold per step."""

    method = "jacobi"

    def _rebuild(self):
        L, o = self._lay, self.ops
        self._rh = o.zeros(L.n + 2 * L.halo)
        self._x2h = o.zeros(L.n + 2 * L.halo)
        self._r2h = o.zeros(L.n + 2 * L.halo)
        self._halo(self._xh)
        o.residual(L.slab, self._xh, L.halo, self.b, self._rh[L.halo:], 0.0, None, 0, self._part, None)
        o.fold(self._gathered(2), 2, L.nch_global, KOP_RESID_INIT, self.sc)
        self._range_valid = False
        self._sync()

    def _enqueue_step(self):
        L, o = self._lay, self.ops
        self._halo(self._xh)
        self._halo(self._rh)
        o.jacobi(L.slab, self.m.inverse_diagonal, self._xh, L.halo, self._rh, L.halo, self.b, self._x2h, L.halo,
                 self._r2h, L.halo, self.sc, self._part, self._rparts)
        o.fold(self._gathered(1), 1, L.nch_global, KOP_RESID, self.sc, rparts=self._rparts, nrp=L.nch,
               rout=self._range)
        self._xh, self._x2h = self._x2h, self._xh
        self._rh, self._r2h = self._r2h, self._rh
        self._range_valid = True
        self._planned += 1


class CgSolver(_SolverBase):
    """Preconditioned CG restarted every restart_len iterations (solvers.py:113-148).

    Per iteration: p halo exchange, q = A p with the p.q partials, alpha
    (fold), the fused x/r update with the r.z and r.r partials and the range
    of x, beta / rho / residual / convergence (fold), p = z + beta p.  All
    scalars stay on the device."""

    method = "cg"

    def _rebuild(self, in_step=False):
        L, o = self._lay, self.ops
        if not hasattr(self, "_ph"):
            self._ph = o.zeros(L.n + 2 * L.halo)
            self._r = o.empty(L.n)
            self._q = o.empty(L.n)
        self._halo(self._xh)
        # r = b - A x, z = p = inv*r, (r.z, r.r) partials
        o.residual(L.slab, self._xh, L.halo, self.b, self._r, self.m.inverse_diagonal, self._ph, L.halo,
                   self._part, self.sc if in_step else None)
        o.fold(self._gathered(2), 2, L.nch_global, KOP_REBUILD_STEP if in_step else KOP_REBUILD_INIT, self.sc)
        self._fresh = True
        if not in_step:
            self._range_valid = False
            self._sync()

    def _enqueue_step(self):
        L, o = self._lay, self.ops
        it = self._planned
        if it > 0 and not self._fresh and it % self.config.restart_len == 0:
            self._rebuild(in_step=True)
        self._fresh = False
        self._halo(self._ph)
        o.spmv(L.slab, self._ph, L.halo, self._q, self._part, self.sc)
        o.fold(self._gathered(1), 1, L.nch_global, KOP_ALPHA, self.sc)
        o.cg_update(L.n, self._ph, L.halo, self._q, self._xh, L.halo, self._r, self.m.inverse_diagonal, self.sc,
                    self._part, self._rparts)
        o.fold(self._gathered(2), 2, L.nch_global, KOP_BETA, self.sc, rparts=self._rparts, nrp=L.nch,
               rout=self._range)
        o.cg_dir(L.n, self._r, self._ph, L.halo, self.m.inverse_diagonal, self.sc)
        self._range_valid = True
        self._planned += 1

    @property
    def r(self):
        return self._r


class GmresSolver(_SolverBase):
    """Restarted GMRES(k), modified Gram-Schmidt + Givens (solvers.py:151-241).

    The Krylov basis lives in HBM (one slab per rank); the dots, the basis
    updates and normalisations are device kernels with device scalars; the
    projected (k+1) x k system and the Givens rotations are host scalars as
    in the reference, read once per iteration (the column of H)."""

    method = "gmres"

    def _host_residual(self, value: float):
        if not math.isfinite(value):
            raise BreakdownError("residual norm is not finite", self.iteration)
        self.residual_norm = value
        self.converged = value <= self.config.tolerance * self.norm_b

    def _residual_norm_dev(self):
        """r = b - A x into self._w; the norm lands in self._out[1] (and sc.res)."""
        L, o = self._lay, self.ops
        self._halo(self._xh)
        o.residual(L.slab, self._xh, L.halo, self.b, self._w, 0.0, None, 0, self._part, None)
        o.fold(self._gathered(2), 2, L.nch_global, KOP_RESID_INIT, self.sc, out=self._out, outoff=1,
               rparts=self._rparts if self._range_valid else None, nrp=L.nch, rout=self._range)

    def _rebuild(self):
        L, o = self._lay, self.ops
        k = self.config.restart_len
        self._ld = L.n + 2 * L.halo
        if getattr(self, "_basis", None) is None or self._basis.numel() != (k + 1) * self._ld:
            self._basis = o.zeros((k + 1) * self._ld)
            self._w = o.empty(L.n)
            self._h = o.zeros(k + 2)
            self._y = o.zeros(k + 1)
        self._x_base = self._xh.clone()
        self._rmat = np.zeros((k + 1, k))
        self._givens = np.zeros((k, 2))
        self._g = np.zeros(k + 1)
        self._inner = 0
        self._cycle_closed = False
        self._residual_norm_dev()
        beta = float(o.read(self._out)[1])
        self._host_residual(beta)
        if beta > 0.0:
            o.div(L.n, self._w, self._basis, L.halo, self._out, 1, None)     # r / beta
            self._g[0] = beta
        else:
            self._cycle_closed = True

    @property
    def basis_size(self) -> int:
        return self._inner + 1 if not self._cycle_closed else 0

    def _finalize_cycle(self):
        L, o = self._lay, self.ops
        j = self._inner
        y = np.zeros(j)
        for row in range(j - 1, -1, -1):
            diag = self._rmat[row, row]
            if diag == 0.0:
                raise BreakdownError("GMRES breakdown: singular projected system", self.iteration)
            y[row] = (self._g[row] - self._rmat[row, row + 1:j] @ y[row + 1:]) / diag
        if j:
            o.write(self._y[:j], y)
        xnew = o.zeros(L.n + 2 * L.halo)
        o.combine(L.n, j, self._basis, L.halo, self._ld, self._y, self._x_base, xnew, L.halo, self._rparts)
        self._xh = xnew
        self._range_valid = True
        self._cycle_closed = True
        self._residual_norm_dev()
        self._host_residual(float(o.read(self._out)[1]))

    def step(self):
        self._check_steppable()
        if self._cycle_closed:
            self._rebuild()
        L, o = self._lay, self.ops
        j = self._inner
        ld = self._ld
        vj = self._basis[j * ld:(j + 1) * ld]
        self._halo(vj)
        o.spmv(L.slab, vj, L.halo, self._w, None, None)
        for i in range(j + 1):
            o.dot(L.n, self._basis, i * ld + L.halo, self._w, 0, self._part, None)
            o.fold(self._gathered(1), 1, L.nch_global, KOP_DOT, None, out=self._h, outoff=i)
            o.subh(L.n, self._basis, i * ld + L.halo, self._w, self._h, i, None)
        o.dot(L.n, self._w, 0, self._w, 0, self._part, None)
        o.fold(self._gathered(1), 1, L.nch_global, KOP_NORM, None, out=self._h, outoff=j + 1)
        hcol = o.read(self._h[:j + 2])                   # the one host round trip of the step
        self._rmat[:j + 1, j] = hcol[:j + 1]
        hnext = float(hcol[j + 1])
        for i in range(j):
            c, s = self._givens[i]
            hi, hk = self._rmat[i, j], self._rmat[i + 1, j]
            self._rmat[i, j] = c * hi + s * hk
            self._rmat[i + 1, j] = -s * hi + c * hk
        denom = float(np.hypot(self._rmat[j, j], hnext))
        if denom == 0.0:
            c, s = 1.0, 0.0
        else:
            c, s = self._rmat[j, j] / denom, hnext / denom
        self._givens[j] = (c, s)
        self._rmat[j, j] = denom
        self._g[j + 1] = -s * self._g[j]
        self._g[j] = c * self._g[j]
        res_est = abs(float(self._g[j + 1]))
        self.iteration += 1
        self._planned = self.iteration
        self._inner = j + 1
        happy = hnext == 0.0
        if not happy:
            o.div(L.n, self._w, self._basis, (j + 1) * ld + L.halo, self._h, j + 1, None)
        if happy or self._inner == self.config.restart_len or res_est <= self.config.tolerance * self.norm_b:
            self._finalize_cycle()
            if happy and not self.converged:
                raise BreakdownError("GMRES happy breakdown with nonzero residual", self.iteration)
        else:
            self._host_residual(res_est)
        return self

    def advance(self, k: int) -> int:
        start = self.iteration
        for _ in range(int(k)):
            if self.converged or self.iteration >= self.config.max_iterations:
                break
            self.step()
        return self.iteration - start


_METHODS = {cls.method: cls for cls in (JacobiSolver, CgSolver, GmresSolver)}
METHOD_NAMES = tuple(_METHODS)


def init(method: str, a, m, b, config: SolveConfig, comm=None, ops=None):
    """Fresh solver at iteration 0 from x = 0 (solvers.py:248-252)."""
    if method not in _METHODS:
        raise ParameterError(f"unknown method {method!r}; expected one of {METHOD_NAMES}")
    return _METHODS[method](a, m, b, config, comm=comm, ops=ops)


def rebuild_from_solution(method: str, a, m, b, x, iteration: int, config: SolveConfig, comm=None, ops=None):
    """Solver state rebuilt from a (possibly lossy) solution vector (solvers.py:260-268)."""
    if method not in _METHODS:
        raise ParameterError(f"unknown method {method!r}; expected one of {METHOD_NAMES}")
    return _METHODS[method](a, m, b, config, x=x, iteration=iteration, comm=comm, ops=ops)


def solve_to_convergence(state, max_iterations: Optional[int] = None):
    """Step until converged or the iteration cap (solvers.py:271-276), BATCH
    iterations per host round trip."""
    cap = state.config.max_iterations if max_iterations is None else max_iterations
    while not state.converged and state.iteration < cap:
        state.advance(min(BATCH, cap - state.iteration))
    return state
