"""Failure injection, rollback and extra-iteration count on the GPU
(north star "Solver harness").

Mirrors simulate.measure_n_prime (simulate.py:443-508) with the GPU solvers
of solvers.py and the checkpoint layer of checkpoint.py: the solver vector
never leaves HBM except as the compressed checkpoint payload.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import checkpoint as ckpt
from . import solvers
from .compressor import CompressorConfig
from .errors import ParameterError


@dataclass(frozen=True)
class NPrimeSample:
    inject_at: int
    recovered_from: int
    n_prime: Optional[int]
    converged: bool


@dataclass(frozen=True)
class NPrimeResult:
    baseline_n: int
    samples: tuple

    def values(self) -> np.ndarray:
        return np.array([s.n_prime if s.n_prime is not None else np.nan for s in self.samples], dtype=np.float64)


def measure_n_prime(method: str, a, m, b, solve_config: solvers.SolveConfig,
                    comp_config: Optional[CompressorConfig], injection_points,
                    ckpt_intvl: Optional[int] = None) -> NPrimeResult:
    """Per-recovery extra iterations from single injected failures (simulate.py:461-508).

    For each injection iteration j the solver runs to j with checkpoints every
    ckpt_intvl iterations, is struck once, recovers from the last image (or
    restarts from scratch if none exists) and runs to convergence; the sample
    is final_iterations - baseline_iterations.  comp_config None selects
    traditional (lossless) checkpoints.
    """
    k = solve_config.ckpt_intvl if ckpt_intvl is None else ckpt_intvl
    if k < 1:
        raise ParameterError("ckpt_intvl must be >= 1")
    baseline = solvers.solve_to_convergence(solvers.init(method, a, m, b, solve_config))
    if not baseline.converged:
        raise ParameterError("failure-free baseline did not converge; fix the setup first")
    base_n = baseline.iteration

    def rebuild(method_, a_, m_, b_, x, iteration, config):
        return solvers.rebuild_from_solution(method_, a_, m_, b_, x, iteration, config)

    store = ckpt.StorageTarget()
    samples = []
    for j in injection_points:
        j = int(j)
        if not 0 < j < base_n:
            raise ParameterError(f"injection point {j} outside (0, baseline {base_n})")
        solver = solvers.init(method, a, m, b, solve_config)
        last_image = None
        while solver.iteration < j and not solver.converged:
            it = solver.iteration
            if it > 0 and it % k == 0:
                if comp_config is None:
                    last_image, _ = ckpt.checkpoint_traditional(solver, store)
                else:
                    last_image, _ = ckpt.checkpoint_lossy(solver, comp_config, store)
            # to the next checkpoint or the failure in one host round trip
            solver.advance(min(k - it % k, j - it))
        if last_image is not None:
            solver, _ = ckpt.recover(last_image, method, a, m, b, solve_config, rebuild=rebuild,
                                     device=solver.x.device)
            recovered_from = last_image.iteration
        else:
            solver = solvers.init(method, a, m, b, solve_config)
            recovered_from = 0
        solvers.solve_to_convergence(solver)
        samples.append(NPrimeSample(inject_at=j, recovered_from=recovered_from,
                                    n_prime=solver.iteration - base_n if solver.converged else None,
                                    converged=solver.converged))
    return NPrimeResult(baseline_n=base_n, samples=tuple(samples))


@dataclass(frozen=True)
class TrialResult:
    baseline_n: int
    final_n: int
    converged: bool
    recovered_from: tuple
    ratios: tuple              # compression ratio (raw bytes / block bytes) of every lossy checkpoint
    t_compress: tuple          # seconds per lossy checkpoint (compress, host wall clock)
    t_decompress: tuple        # seconds per recovery (decode)
    seconds: float             # whole trial

    @property
    def n_prime(self):
        return self.final_n - self.baseline_n if self.converged else None


def multi_failure_trial(method, a, m, b, solve_config: solvers.SolveConfig, comp_config: Optional[CompressorConfig],
                        failures, ckpt_intvl: Optional[int] = None, baseline_n: Optional[int] = None,
                        comm=None, block_version: Optional[int] = None) -> TrialResult:
    """One run with several injected failures (BASELINE.json config 3: failures
    at iterations 100 and 300).  A checkpoint is taken every k iterations
    (not again at the iteration just recovered to); when the solver first
    reaches a listed iteration its state is lost and rebuilt from the last
    image (from scratch if none).  N' = final - baseline iterations.  The
    same protocol as tests/golden/make_config_golden.py runs on the real
    reference (simulate.measure_n_prime, simulate.py:461-508, with more than
    one failure per run).  block_version: the image's block format (None: the
    checkpoint layer's default, v3; 1: the reference's bytes and ratios)."""
    import time
    k = solve_config.ckpt_intvl if ckpt_intvl is None else ckpt_intvl
    if k < 1:
        raise ParameterError("ckpt_intvl must be >= 1")
    if baseline_n is None:
        base = solvers.solve_to_convergence(solvers.init(method, a, m, b, solve_config, comm=comm))
        if not base.converged:
            raise ParameterError("failure-free baseline did not converge; fix the setup first")
        baseline_n = base.iteration
    t0 = time.perf_counter()
    store = ckpt.StorageTarget()
    solver = solvers.init(method, a, m, b, solve_config, comm=comm)
    pending = sorted(int(f) for f in failures)
    last, recovered_at = None, None
    recs, ratios, tc, td = [], [], [], []

    def rebuild(method_, a_, m_, b_, x, iteration, config):
        return solvers.rebuild_from_solution(method_, a_, m_, b_, x, iteration, config, comm=comm)

    while not solver.converged and solver.iteration < solve_config.max_iterations:
        it = solver.iteration
        if pending and it == pending[0]:
            pending.pop(0)
            if last is None:
                solver = solvers.init(method, a, m, b, solve_config, comm=comm)
            else:
                solver, cost = ckpt.recover(last, method, a, m, b, solve_config, rebuild=rebuild,
                                            device=solver.x.device)
                td.append(cost.t_decompress)
            recs.append(solver.iteration)
            recovered_at = solver.iteration
            continue
        if it > 0 and it % k == 0 and it != recovered_at:
            if comp_config is None:
                last, cost = ckpt.checkpoint_traditional(solver, store)
            else:
                last, cost = ckpt.checkpoint_lossy(solver, comp_config, store, block_version=block_version)
                ratios.append(solver.x.numel() * 8 / len(last.payload))
                tc.append(cost.t_compress)
        nxt = [it - it % k + k]
        if pending:
            nxt.append(pending[0])
        solver.advance(max(1, min(nxt) - it))
    return TrialResult(baseline_n=baseline_n, final_n=solver.iteration, converged=solver.converged,
                       recovered_from=tuple(recs), ratios=tuple(ratios), t_compress=tuple(tc),
                       t_decompress=tuple(td), seconds=time.perf_counter() - t0)


# --- GPU workload for the reference's Poisson-failure trials (simulate.py:207-384) ----
#
# The event loop itself is the reference's: lossyckpt.simulate.run_trial(config,
# seed, workload=GpuSolverWorkload(config)) accepts any workload with this
# protocol, so it is not re-implemented here (the event loop
# has no data-parallel work).

def build_problem(problem: str, device="cuda"):
    """(matrix, preconditioner, b) on the device (simulate.py:145-158 + the 3-D configs)."""
    import torch
    kind, _, arg = problem.partition(":")
    try:
        size = int(arg)
    except ValueError:
        raise ParameterError(f"malformed problem spec {problem!r}") from None
    if kind == "poisson2d":
        a, b = solvers.generate_poisson2d(size, device=device)
    elif kind == "poisson1d":
        if size < 1:
            raise ParameterError("n must be >= 1")
        a = solvers.StencilMatrix(size, 1, 1, 2.0, -1.0, -1.0)
        b = torch.ones(size, dtype=torch.float64, device=device)
    elif kind == "laplacian3d":
        a = solvers.generate_laplacian3d(size)
        b = torch.ones(a.n_rows, dtype=torch.float64, device=device)
    elif kind == "convdiff3d":
        a = solvers.generate_convdiff3d(size)
        b = torch.ones(a.n_rows, dtype=torch.float64, device=device)
    else:
        raise ParameterError(f"unknown problem kind {kind!r}")
    return a, solvers.jacobi_preconditioner(a), b


class GpuSolverWorkload:
    """A GPU iterative solver driven through the checkpoint layer.

    Same protocol as the reference's _SolverWorkload (simulate.py:207-270):
    iteration, converged, diverged, remaining(), advance(n), capture(now),
    recovery_cost(image), restore(image), reset().  `config` is the
    reference's SimConfig (simulate.py:62-120; duck-typed: method, problem,
    tolerance, max_iterations, effective_restart_len, ckpt_intvl, policy,
    compressor_config, bandwidths and injected durations); hand the workload
    to the reference's own run_trial(config, seed, workload=...).
    """

    def __init__(self, config, problem=None):
        self.a, self.m, self.b = problem if problem is not None else build_problem(config.problem)
        self.solve_config = solvers.SolveConfig(
            tolerance=config.tolerance, max_iterations=config.max_iterations,
            restart_len=config.effective_restart_len, ckpt_intvl=config.ckpt_intvl)
        self._config = config
        self.store = ckpt.StorageTarget(write_bandwidth=config.write_bandwidth,
                                        read_bandwidth=config.read_bandwidth)
        self.diverged = False
        self.solver = solvers.init(config.method, self.a, self.m, self.b, self.solve_config)

    @property
    def iteration(self) -> int:
        return self.solver.iteration

    @property
    def converged(self) -> bool:
        return self.solver.converged

    def remaining(self):
        return None

    def advance(self, n: int) -> int:
        done = 0
        cap = self.solve_config.max_iterations
        while done < n and not self.solver.converged and self.solver.iteration < cap:
            done += self.solver.advance(min(n - done, solvers.BATCH))
        if not self.solver.converged and self.solver.iteration >= cap:
            self.diverged = True
        return done

    def capture(self, now: float = 0.0):
        if self._config.policy == "lossy":
            image, cost = ckpt.checkpoint_lossy(self.solver, self._config.compressor_config, self.store,
                                                created_at=now, t_comp_override=self._config.t_comp,
                                                commit=False)
        else:
            image, cost = ckpt.checkpoint_traditional(self.solver, self.store, created_at=now, commit=False)
        duration = self._config.t_ckpt if self._config.t_ckpt is not None else cost.total
        return image, duration

    def recovery_cost(self, image) -> float:
        if self._config.t_rc is not None:
            return self._config.t_rc
        if image is None:
            return 0.0
        t_read = self.store.read_time(image.nbytes)
        t_dec = self._config.t_decomp if image.kind == ckpt.PAYLOAD_LOSSY else 0.0
        return t_read + t_dec

    def restore(self, image) -> None:
        def rebuild(method_, a_, m_, b_, x, iteration, config):
            return solvers.rebuild_from_solution(method_, a_, m_, b_, x, iteration, config)

        self.solver, _ = ckpt.recover(image, self._config.method, self.a, self.m, self.b, self.solve_config,
                                      t_decomp_override=0.0, rebuild=rebuild, device=self.solver.x.device)

    def reset(self) -> None:
        self.solver = solvers.init(self._config.method, self.a, self.m, self.b, self.solve_config)
