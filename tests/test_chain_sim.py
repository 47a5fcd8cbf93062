"""Host simulation of the chunked exact chain (product header lc_chain.cuh
compiled with g++): the superset flag tracker + replay reproduces the step-by-step
offset map of every chunk, and the composed maps predict every chunk start of
the sequential reference chain (compressor.py:319-355) -- sequential and
tree-ordered composition (the GPU's in-tile scan + tile scan order)."""

import shutil

import numpy as np
import pytest

from tests.cpu import chain_sim_run as cs


@pytest.fixture(scope="module")
def sim():
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    return cs.build()


def test_tracker_and_prediction(sim):
    for name, (x, ebs) in cs.vectors(seed=0, n=1 << 15).items():
        vr = float(x.max() - x.min())
        for ebr in ebs:
            for mode in (0, 1):
                bad, first, changes, flagged, chunks = cs.predict(sim, x, ebr * vr, mode=mode)
                assert flagged >= 0, (name, ebr, mode)         # tracker == step-by-step map
                if name != "ints":                              # integer data may need a relaunch
                    assert bad == 0, (name, ebr, mode, first)


def test_golden_vectors(sim, golden):
    # jac190_r6 / edge_0 carry escapes: the simulator has no escape anchors
    # (the GPU path does), so only the tracker is checked there
    for key in ("jac190_r4", "jac190_r6", "sine_r6", "edge_0", "crit6_2"):
        x = golden[str(golden[key + "/x"])]
        mode, param, nbh = golden[key + "/cfg"]
        vr = float(x.max() - x.min())
        eb = float(param) if int(mode) == 0 else float(param) * vr
        for m in (0, 1):
            bad, first, changes, flagged, chunks = cs.predict(sim, x, eb, nbh=int(nbh), mode=m)
            assert flagged >= 0, (key, m)
            if key not in ("jac190_r6", "edge_0"):
                assert bad == 0, (key, m, first)
