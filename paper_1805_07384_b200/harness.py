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
            solver.step()
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


# --- Poisson-failure trials over a GPU solver workload (simulate.py:39-384) ----------

import math  # noqa: E402
from dataclasses import dataclass as _dc  # noqa: E402

_POLICIES = ("traditional", "lossy", "none")


@_dc(frozen=True)
class FailureProcess:
    """Poisson failures: i.i.d. exponential inter-arrival times with rate lam (simulate.py:41-57)."""

    lam: float
    rng_seed: int

    def __post_init__(self):
        if self.lam < 0:
            raise ParameterError("failure rate must be non-negative")

    def arrivals(self):
        rng = np.random.default_rng(self.rng_seed)
        scale = 1.0 / self.lam if self.lam > 0 else math.inf

        def draw() -> float:
            return float(rng.exponential(scale)) if self.lam > 0 else math.inf

        return draw


@_dc(frozen=True)
class SimConfig:
    """Reproducible simulation setup for GPU solver workloads (simulate.py:60-121).

    Problems: poisson2d:M, poisson1d:N (the reference's) and laplacian3d:M,
    convdiff3d:M (BASELINE.json configs 3-5).  The reference's synthetic
    workload is host bookkeeping only and not reproduced here.
    """

    method: str = "jacobi"
    problem: str = "poisson2d:64"
    policy: str = "traditional"
    ckpt_intvl: int = 100
    t_it: float = 1.0
    lam: float = 0.0
    seed: int = 0
    trials: int = 1
    max_time: float = math.inf
    tolerance: float = 1e-8
    max_iterations: int = 200_000
    restart_len: Optional[int] = None
    compressor_config: Optional[CompressorConfig] = None
    t_ckpt: Optional[float] = None
    t_rc: Optional[float] = None
    t_comp: float = 0.0
    t_decomp: float = 0.0
    write_bandwidth: Optional[float] = None
    read_bandwidth: Optional[float] = None
    failures_during_ckpt: bool = True

    def __post_init__(self):
        if self.method not in solvers.METHOD_NAMES:
            raise ParameterError(f"unknown method {self.method!r}")
        if self.policy not in _POLICIES:
            raise ParameterError(f"unknown policy {self.policy!r}")
        if self.trials < 1 or self.ckpt_intvl < 1 or self.t_it <= 0 or self.lam < 0:
            raise ParameterError("trials, ckpt_intvl must be >= 1; t_it > 0; lam >= 0")
        if self.policy == "lossy" and self.compressor_config is None:
            raise ParameterError("real lossy policy needs a compressor_config")

    @property
    def effective_restart_len(self) -> int:
        return self.ckpt_intvl if self.restart_len is None else self.restart_len


@_dc(frozen=True)
class TrialReport:
    """Exact bookkeeping of one trial in simulated time units (simulate.py:124-142)."""

    seed: int
    converged: bool
    truncated: bool
    diverged: bool
    total_time: float
    productive_time: float
    ckpt_time: float
    rc_time: float
    rollback_time: float
    iterations_final: int
    iterations_executed: int
    n_failures: int
    n_checkpoints: int
    n_checkpoints_voided: int
    n_recoveries: int
    n_lossy_recoveries: int


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
    recovery_cost(image), restore(image), reset().  It can also be handed to
    the reference's own run_trial(config, seed, workload=...).
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
            self.solver.step()
            done += 1
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


def run_trial(config: SimConfig, seed: int, workload=None) -> TrialReport:
    """One trial: iterate, checkpoint every ckpt_intvl iterations, inject Poisson
    failures, recover from the last image (simulate.py:277-384, same event order)."""
    if workload is None:
        workload = GpuSolverWorkload(config)
    draw = FailureProcess(config.lam, seed).arrivals()
    k = config.ckpt_intvl
    interruptible = config.failures_during_ckpt and config.lam > 0
    t = 0.0
    next_fail = draw()
    ckpt_time = rc_time = fragments = 0.0
    executed = 0
    n_failures = n_ckpts = n_voided = n_recoveries = n_lossy = 0
    last_image = None
    last_ckpt_iter = -1
    pending_failure = False
    truncated = False
    while True:
        if workload.converged or workload.diverged:
            break
        if t >= config.max_time:
            truncated = True
            break
        if pending_failure:
            pending_failure = False
            n_failures += 1
            next_fail = t + draw()
            while True:                      # recovery, possibly struck by further failures
                cost = workload.recovery_cost(last_image)
                if interruptible and next_fail < t + cost:
                    rc_time += next_fail - t
                    t = next_fail
                    n_failures += 1
                    next_fail = t + draw()
                    if t >= config.max_time:
                        truncated = True
                        break
                    continue
                rc_time += cost
                t += cost
                if last_image is not None:
                    workload.restore(last_image)
                    if config.policy == "lossy":
                        n_lossy += 1
                else:
                    workload.reset()
                last_ckpt_iter = -1
                n_recoveries += 1
                break
            if truncated:
                break
            continue
        i = workload.iteration
        if config.policy != "none" and i > 0 and i % k == 0 and i != last_ckpt_iter:
            image, cost = workload.capture(t)
            if interruptible and next_fail < t + cost:
                ckpt_time += next_fail - t       # in-flight image is voided
                t = next_fail
                n_voided += 1
                pending_failure = True
                continue
            ckpt_time += cost
            t += cost
            last_image = image
            last_ckpt_iter = i
            n_ckpts += 1
            continue
        if config.lam > 0:
            headroom = (next_fail - t) / config.t_it
            if headroom < 1.0:
                frag = max(0.0, next_fail - t)
                fragments += frag
                t += frag
                pending_failure = True
                continue
            budget = int(headroom)
        else:
            budget = config.max_iterations + 1
        n = min(budget, (k - i % k) if config.policy != "none" else budget)
        rem = workload.remaining()
        if rem is not None:
            n = min(n, rem)
        done = workload.advance(n)
        executed += done
        t += done * config.t_it
    final_iter = workload.iteration
    productive = final_iter * config.t_it
    rollback = (executed - final_iter) * config.t_it + fragments
    return TrialReport(seed=seed, converged=bool(workload.converged), truncated=truncated,
                       diverged=bool(workload.diverged), total_time=t, productive_time=productive,
                       ckpt_time=ckpt_time, rc_time=rc_time, rollback_time=rollback,
                       iterations_final=final_iter, iterations_executed=executed, n_failures=n_failures,
                       n_checkpoints=n_ckpts, n_checkpoints_voided=n_voided, n_recoveries=n_recoveries,
                       n_lossy_recoveries=n_lossy)
