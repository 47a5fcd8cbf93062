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
