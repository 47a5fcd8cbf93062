"""Golden Poisson-failure trials from the REAL reference (simulate.run_trial with
its own _SolverWorkload), for the GPU harness's run_trial/GpuSolverWorkload.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_trial_golden.py

Writes tests/golden/trial_golden.json: per case the SimConfig fields and the
TrialReport the reference produced.  Checkpoint/recovery durations are injected
so the event sequence is deterministic.
"""

import dataclasses
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from lossyckpt import simulate  # noqa: E402
from lossyckpt.compressor import CompressorConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "trial_golden.json")
CASES = [
    dict(method="jacobi", problem="poisson2d:24", policy="lossy", ckpt_intvl=20, lam=1 / 400, t_ckpt=3.0,
         t_rc=5.0, tolerance=1e-6, seed=7, eb_rel=1e-4),
    dict(method="jacobi", problem="poisson1d:60", policy="traditional", ckpt_intvl=25, lam=1 / 900, t_ckpt=2.0,
         t_rc=4.0, tolerance=1e-6, seed=11, eb_rel=None),
    dict(method="cg", problem="poisson2d:24", policy="lossy", ckpt_intvl=10, lam=1 / 60, t_ckpt=2.0,
         tolerance=1e-8, seed=3, eb_rel=1e-5),
    dict(method="gmres", problem="poisson2d:16", policy="lossy", ckpt_intvl=10, lam=1 / 25, t_ckpt=1.0,
         tolerance=1e-8, seed=5, eb_rel=1e-5),
]
out = []
for c in CASES:
    kw = {k: v for k, v in c.items() if k not in ("eb_rel",)}
    if c["eb_rel"] is not None:
        kw["compressor_config"] = CompressorConfig.value_range_relative(c["eb_rel"])
    cfg = simulate.SimConfig(**kw)
    rep = simulate.run_trial(cfg, c["seed"])
    out.append({"config": c, "report": dataclasses.asdict(rep)})
    print(c["method"], c["problem"], dataclasses.asdict(rep), flush=True)
json.dump(out, open(OUT, "w"), indent=1)
print("wrote", OUT)
