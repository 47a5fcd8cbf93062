"""Profiling driver for BASELINE.json config-5 data: the x slab of CG on the 3-D
Laplacian side^3 (b ~ U(-1,1) seed 3) after `iters` iterations, compressed at rel
eb and decompressed (one warm-up + one measured round trip; device phases printed).

    python profiles/prof_cfg5.py [side=512] [iters=100] [eb=1e-5]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_07384_b200 import _native, solvers  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
eb = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-5
a = solvers.generate_laplacian3d(side)
b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, a.n_rows)).cuda()
s = solvers.init("cg", a, solvers.jacobi_preconditioner(a), b,
                 solvers.SolveConfig(tolerance=1e-8, restart_len=25, ckpt_intvl=25))
s.advance(iters)
n = a.n_rows
ctx = _native.context(0)
L = ctx.lib
out = torch.empty(n, dtype=torch.float64, device="cuda")
vp = ctypes.c_void_p
for rep in range(2):
    res, bnd = _native.LcResult(), _native.LcBounds()
    rc = L.lc_compress_ranged_f64(ctx.h, s.x.data_ptr(), n, 1, eb, 32768, 0, s.x_range.data_ptr(),
                                  ctypes.byref(res), ctypes.byref(bnd))
    assert rc == 0, ctx.error()
    tc = L.lc_last_device_ms(ctx.h)
    ph = (ctypes.c_double * 8)()
    L.lc_phase_ms(ctx.h, ph, 8)
    cph = [round(ph[i], 4) for i in range(4)]
    pay, cl, ei, ev = vp(), vp(), vp(), vp()
    L.lc_result_device(ctx.h, ctypes.byref(pay), ctypes.byref(cl), ctypes.byref(ei), ctypes.byref(ev))
    used = ctypes.c_int64()
    rc = L.lc_decompress_f64(ctx.h, n, bnd.eb_abs, bnd.first_value, cl, res.n_symbols, pay, res.payload_bytes,
                             res.payload_bits, ei, ev, res.n_esc, 1, out.data_ptr(), 1, ctypes.byref(used))
    assert rc == 0, ctx.error()
    td = L.lc_last_device_ms(ctx.h)
    L.lc_phase_ms(ctx.h, ph, 8)
    dph = [round(ph[i], 4) for i in range(4, 8)]
err = float((out - s.x).abs().max()) / bnd.eb_abs
print("n", n, "eb", eb, "compress_ms", round(tc, 3), cph, "decompress_ms", round(td, 3), dph,
      "symbols", res.used_symbols, "max_len", res.max_len, "bits/sym", res.payload_bits / (n - 1),
      "relaunches", res.relaunches, "exact_chunks", L.lc_ctx_get_stat(ctx.h, 4), "err/eb", err)
