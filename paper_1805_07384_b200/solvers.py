"""On-GPU solver harness (north star "Solver harness").

Mirrors lossyckpt/solvers.py (SolveConfig, JacobiSolver, CgSolver,
GmresSolver, init, rebuild_from_solution, solve_to_convergence; solvers.py:
23-276) for the constant-coefficient stencil matrices of BASELINE.json's
configs, with state vectors as torch CUDA float64 tensors and every vector
operation in the hand-written kernels of csrc/lc_solver.cu (stencil SpMV,
fused Jacobi step, residual, dot, axpy) through the C ABI.

Arithmetic follows the reference operation by operation: y = A x is
accumulated in CSR column order with unfused multiply/add (bit-identical to
sparse.py:21-28), updates are one rounded multiply and one rounded add as in
the numpy expressions, so Jacobi iterates are bit-identical to the
reference.  Dot products and norms use a fixed-order parallel reduction
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


def _residual(a, x, b, r) -> float:
    ctx = _ctx(x)
    st = a.abi()
    out = ctypes.c_double()
    _check(ctx, ctx.lib.lc_residual_f64(ctx.h, ctypes.addressof(st), x.data_ptr(), b.data_ptr(), r.data_ptr(),
                                        None, ctypes.byref(out)), "residual")
    return math.sqrt(out.value)


def _scaled(alpha: float, x):
    """alpha * x as a new vector (one rounded multiply per element)."""
    import torch
    out = torch.zeros_like(x)
    axpy(alpha, x, out)                  # 0 + RN(alpha*x) == RN(alpha*x)
    return out


# --- solvers ---------------------------------------------------------------------

class _SolverBase:
    method = "?"

    def __init__(self, a: StencilMatrix, m: DiagonalPreconditioner, b, config: SolveConfig,
                 x=None, iteration: int = 0):
        import torch
        b = torch.as_tensor(b, dtype=torch.float64)
        if not b.is_cuda:
            b = b.cuda()
        b = b.contiguous().reshape(-1)
        if a.n_rows != b.numel():
            raise DimensionMismatchError("matrix and right-hand side sizes differ")
        if m.n != a.n_rows:
            raise DimensionMismatchError("preconditioner size differs from matrix")
        if x is None:
            x = torch.zeros_like(b)
        else:
            x = torch.as_tensor(x, dtype=torch.float64).to(b.device).reshape(-1).clone()
            if x.numel() != a.n_rows:
                raise DimensionMismatchError("initial guess size differs from matrix")
        if iteration < 0:
            raise ParameterError("iteration index must be non-negative")
        self.a, self.m, self.b = a, m, b
        self.config = config
        self.x = x
        self.iteration = iteration
        self.norm_b = math.sqrt(dot(b, b))
        self.residual_norm = math.inf
        self.converged = False
        self._rebuild()

    def _rebuild(self):
        raise NotImplementedError

    def _set_residual(self, value: float):
        if not math.isfinite(value):
            raise BreakdownError("residual norm is not finite", self.iteration)
        self.residual_norm = value
        self.converged = value <= self.config.tolerance * self.norm_b

    def _check_steppable(self):
        if self.converged:
            raise ParameterError("step() called on a converged solver")
        if self.iteration >= self.config.max_iterations:
            raise ParameterError("step() called at the iteration cap")

    def step(self):
        raise NotImplementedError


class JacobiSolver(_SolverBase):
    """x <- x + M^-1 (b - A x) (solvers.py:92-110); one fused kernel per step."""

    method = "jacobi"

    def _rebuild(self):
        import torch
        self._r = torch.empty_like(self.x)
        self._x2 = torch.empty_like(self.x)
        self._r2 = torch.empty_like(self.x)
        self._set_residual(_residual(self.a, self.x, self.b, self._r))

    def step(self):
        self._check_steppable()
        ctx = _ctx(self.x)
        st = self.a.abi()
        out = ctypes.c_double()
        _check(ctx, ctx.lib.lc_jacobi_step_f64(ctx.h, ctypes.addressof(st), float(self.m.inverse_diagonal),
                                               self.x.data_ptr(), self._r.data_ptr(), self.b.data_ptr(),
                                               self._x2.data_ptr(), self._r2.data_ptr(), None,
                                               ctypes.byref(out)), "jacobi step")
        self.x, self._x2 = self._x2, self.x
        self._r, self._r2 = self._r2, self._r
        self.iteration += 1
        self._set_residual(math.sqrt(out.value))
        return self


class CgSolver(_SolverBase):
    """Preconditioned CG restarted every restart_len iterations (solvers.py:113-148)."""

    method = "cg"

    def _rebuild(self):
        import torch
        self.r = torch.empty_like(self.x)
        rn = _residual(self.a, self.x, self.b, self.r)
        self.z = _scaled(self.m.inverse_diagonal, self.r)
        self.p = self.z.clone()
        self.rho = dot(self.r, self.z)
        self._fresh = True
        self._set_residual(rn)

    def step(self):
        self._check_steppable()
        if self.iteration > 0 and not self._fresh and self.iteration % self.config.restart_len == 0:
            self._rebuild()
        self._fresh = False
        q = spmv(self.a, self.p)
        pq = dot(self.p, q)
        if self.rho == 0.0 or pq == 0.0:
            raise BreakdownError("CG breakdown: zero curvature or zero rho", self.iteration)
        alpha = self.rho / pq
        axpy(alpha, self.p, self.x)                    # x + alpha*p
        axpy(-alpha, q, self.r)                        # r - alpha*q
        self.z = _scaled(self.m.inverse_diagonal, self.r)
        rho_new = dot(self.r, self.z)
        p_scaled = _scaled(rho_new / self.rho, self.p)
        axpy(1.0, self.z, p_scaled)                    # z + beta*p
        self.p = p_scaled
        self.rho = rho_new
        self.iteration += 1
        self._set_residual(math.sqrt(dot(self.r, self.r)))
        return self


class GmresSolver(_SolverBase):
    """Restarted GMRES(k), modified Gram-Schmidt + Givens (solvers.py:151-241).

    The Krylov basis lives in HBM; the projected system (k x k) and the Givens
    rotations are host scalars as in the reference.
    """

    method = "gmres"

    def _rebuild(self):
        import torch
        k = self.config.restart_len
        n = self.a.n_rows
        self._x_base = self.x.clone()
        self._basis = torch.zeros((k + 1, n), dtype=torch.float64, device=self.x.device)
        self._rmat = np.zeros((k + 1, k))
        self._givens = np.zeros((k, 2))
        self._g = np.zeros(k + 1)
        self._inner = 0
        self._cycle_closed = False
        r = torch.empty_like(self.x)
        beta = _residual(self.a, self.x, self.b, r)
        self._set_residual(beta)
        if beta > 0.0:
            torch.div(r, beta, out=self._basis[0])      # r / beta, one rounded division per element
            self._g[0] = beta
        else:
            self._cycle_closed = True

    @property
    def basis_size(self) -> int:
        return self._inner + 1 if not self._cycle_closed else 0

    def _finalize_cycle(self):
        import torch
        j = self._inner
        y = np.zeros(j)
        for row in range(j - 1, -1, -1):
            diag = self._rmat[row, row]
            if diag == 0.0:
                raise BreakdownError("GMRES breakdown: singular projected system", self.iteration)
            y[row] = (self._g[row] - self._rmat[row, row + 1:j] @ y[row + 1:]) / diag
        x = self._x_base.clone()
        for i in range(j):                              # x_base + sum_i y_i * basis_i
            axpy(float(y[i]), self._basis[i], x)
        self.x = x
        self._cycle_closed = True
        r = torch.empty_like(self.x)
        self._set_residual(_residual(self.a, self.x, self.b, r))

    def step(self):
        self._check_steppable()
        if self._cycle_closed:
            self._rebuild()
        j = self._inner
        w = spmv(self.a, self._basis[j])
        for i in range(j + 1):
            hij = dot(self._basis[i], w)
            axpy(-hij, self._basis[i], w)
            self._rmat[i, j] = hij
        hnext = math.sqrt(dot(w, w))
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
        self._inner = j + 1
        happy = hnext == 0.0
        if not happy:
            import torch
            torch.div(w, hnext, out=self._basis[j + 1])
        if happy or self._inner == self.config.restart_len or res_est <= self.config.tolerance * self.norm_b:
            self._finalize_cycle()
            if happy and not self.converged:
                raise BreakdownError("GMRES happy breakdown with nonzero residual", self.iteration)
        else:
            self._set_residual(res_est)
        return self


_METHODS = {cls.method: cls for cls in (JacobiSolver, CgSolver, GmresSolver)}
METHOD_NAMES = tuple(_METHODS)


def init(method: str, a, m, b, config: SolveConfig):
    """Fresh solver at iteration 0 from x = 0 (solvers.py:248-252)."""
    if method not in _METHODS:
        raise ParameterError(f"unknown method {method!r}; expected one of {METHOD_NAMES}")
    return _METHODS[method](a, m, b, config)


def rebuild_from_solution(method: str, a, m, b, x, iteration: int, config: SolveConfig):
    """Solver state rebuilt from a (possibly lossy) solution vector (solvers.py:260-268)."""
    if method not in _METHODS:
        raise ParameterError(f"unknown method {method!r}; expected one of {METHOD_NAMES}")
    return _METHODS[method](a, m, b, config, x=x, iteration=iteration)


def solve_to_convergence(state, max_iterations: Optional[int] = None):
    """Step until converged or the iteration cap (solvers.py:271-276)."""
    cap = state.config.max_iterations if max_iterations is None else max_iterations
    while not state.converged and state.iteration < cap:
        state.step()
    return state
