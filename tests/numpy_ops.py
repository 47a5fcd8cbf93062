"""CPU double of paper_1805_07384_b200.solvers.DeviceOps (TEST INFRASTRUCTURE).

Same interface and semantics as the lc_krylov.cu kernels -- slab stencil rows
in CSR column order, per-4096-element chunk partials over the GLOBAL vector,
one fixed fold, device-status gating, the lc_kscalars block -- in numpy on
torch CPU tensors, so the slab-sharding host logic (halo exchange, partial
all-gather, batching, restarts) runs under gloo at world size 2 on a machine
without a GPU (tests/test_sharded_solver.py).  The product never uses it."""

import math

import numpy as np
import torch

from paper_1805_07384_b200 import solvers as S

CH = S.CHUNK


def _np(t, off=0, n=None):
    a = t.numpy()
    return a[off:] if n is None else a[off:off + n]


class NumpyOps:
    def __init__(self):
        self.device = torch.device("cpu")

    # storage
    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def as_vector(self, v):
        return torch.as_tensor(v, dtype=torch.float64).reshape(-1).contiguous().clone()

    def scalars(self):
        return torch.zeros(10, dtype=torch.float64)

    def range_record(self):
        return torch.zeros(4, dtype=torch.float64)

    def set_scalars(self, sc, **fields):
        s = S.LcKScalars()
        for k, v in fields.items():
            setattr(s, k, v)
        sc.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.float64))

    def get_scalars(self, sc):
        return S.LcKScalars.from_buffer_copy(sc.numpy().tobytes())

    def _put(self, sc, s):
        sc.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.float64))

    def read(self, t):
        return t.numpy().copy()

    def write(self, dst, host_values):
        dst.copy_(torch.as_tensor(np.asarray(host_values, dtype=np.float64)))

    def _stopped(self, sc):
        return sc is not None and self.get_scalars(sc).status != S.KS_RUNNING

    # helpers
    @staticmethod
    def _rows(slab, v, off):
        st = slab.st
        nx, ny, nz, plane = st.nx, st.ny, st.nz, st.nx * st.ny
        n = plane * slab.nzl
        k = np.arange(n)
        lz, rem = np.divmod(k, plane)
        iy, ix = np.divmod(rem, nx)
        iz = slab.z0 + lz
        acc = np.zeros(n)
        for mask, shift, coef in ((iz > 0, -plane, st.zm), (iy > 0, -nx, st.ym), (ix > 0, -1, st.xm),
                                  (np.ones(n, bool), 0, st.c), (ix < nx - 1, 1, st.xp),
                                  (iy < ny - 1, nx, st.yp), (iz < nz - 1, plane, st.zp)):
            idx = k[mask]
            acc[mask] = acc[mask] + coef * v[off + idx + shift]
        return acc

    @staticmethod
    def _chunks(v):
        n = v.size
        return np.array([np.sum(v[c:c + CH]) for c in range(0, n, CH)])

    def _range(self, x, rparts):
        if rparts is None:
            return
        rp = rparts.numpy().reshape(-1, 6)            # vmin, vmax, maxstep, first, last, nonfinite
        for i, c in enumerate(range(0, x.size, CH)):
            seg = x[c:c + CH]
            rp[i, 0], rp[i, 1] = seg.min(), seg.max()
            rp[i, 2] = np.max(np.abs(np.diff(seg))) if seg.size > 1 else 0.0
            rp[i, 3], rp[i, 4] = seg[0], seg[-1]
            rp[i, 5] = float(not np.all(np.isfinite(seg)))

    # kernels
    def spmv(self, slab, vh, off, y, part, sc):
        if self._stopped(sc):
            return
        v = vh.numpy()
        yv = self._rows(slab, v, off)
        _np(y, 0, yv.size)[:] = yv
        if part is not None:
            p = self._chunks(v[off:off + yv.size] * yv)
            _np(part, 0, p.size)[:] = p

    def residual(self, slab, xh, off, b, r, inv, z, zoff, part, sc_gate):
        if self._stopped(sc_gate):
            return
        rv = _np(b) - self._rows(slab, xh.numpy(), off)
        n = rv.size
        _np(r, 0, n)[:] = rv
        pp = _np(part, 0, 2 * (-(-n // CH))).reshape(-1, 2)
        if z is not None:
            zv = inv * rv
            _np(z, zoff, n)[:] = zv
            pp[:, 0] = self._chunks(rv * zv)
        else:
            pp[:, 0] = 0.0
        pp[:, 1] = self._chunks(rv * rv)

    def cg_update(self, n, p, poff, q, x, xoff, r, inv, sc, part, rparts):
        if self._stopped(sc):
            return
        alpha = self.get_scalars(sc).alpha
        xv = _np(x, xoff, n)
        xv[:] = xv + alpha * _np(p, poff, n)
        rv = _np(r, 0, n)
        rv[:] = rv - alpha * _np(q, 0, n)
        pp = _np(part, 0, 2 * (-(-n // CH))).reshape(-1, 2)
        pp[:, 0] = self._chunks(rv * (inv * rv))
        pp[:, 1] = self._chunks(rv * rv)
        self._range(xv, rparts)

    def cg_dir(self, n, r, p, poff, inv, sc):
        if self._stopped(sc):
            return
        beta = self.get_scalars(sc).beta
        pv = _np(p, poff, n)
        pv[:] = inv * _np(r, 0, n) + beta * pv

    def jacobi(self, slab, inv, xh, xoff, rh, roff, b, x2, x2off, r2, r2off, sc, part, rparts):
        n = slab.st.nx * slab.st.ny * slab.nzl
        if self._stopped(sc):
            _np(x2, x2off, n)[:] = _np(xh, xoff, n)
            _np(r2, r2off, n)[:] = _np(rh, roff, n)
            return
        xn = xh.numpy() + inv * rh.numpy()            # neighbours' new x from (x, r), halos included
        rv = _np(b) - self._rows(slab, xn, xoff)
        _np(x2, x2off, n)[:] = xn[xoff:xoff + n]
        _np(r2, r2off, n)[:] = rv
        p = self._chunks(rv * rv)
        _np(part, 0, p.size)[:] = p
        self._range(xn[xoff:xoff + n], rparts)

    def dot(self, n, a, aoff, b, boff, part, sc):
        if self._stopped(sc):
            return
        p = self._chunks(_np(a, aoff, n) * _np(b, boff, n))
        _np(part, 0, p.size)[:] = p

    def subh(self, n, x, xoff, y, h, hoff, sc):
        yv = _np(y, 0, n)
        yv[:] = yv - h.numpy()[hoff] * _np(x, xoff, n)

    def div(self, n, x, y, yoff, d, doff, sc):
        _np(y, yoff, n)[:] = _np(x, 0, n) / d.numpy()[doff]

    def combine(self, n, j, basis, boff, ld, yv, xbase, x, xoff, rparts):
        bv, yy = basis.numpy(), yv.numpy()
        t = yy[0] * bv[boff:boff + n] if j > 0 else None
        for i in range(1, j):
            t = t + yy[i] * bv[i * ld + boff:i * ld + boff + n]
        xb = _np(xbase, boff, n)
        out = xb + t if j > 0 else xb.copy()
        _np(x, xoff, n)[:] = out
        self._range(out, rparts)

    def fold(self, part, width, nch, op, sc, out=None, outoff=0, rparts=None, nrp=0, rout=None):
        s = self.get_scalars(sc) if sc is not None else None
        if op in (S.KOP_ALPHA, S.KOP_BETA, S.KOP_REBUILD_STEP, S.KOP_RESID) and s.status != S.KS_RUNNING:
            return
        pp = part.numpy()[:width * nch].reshape(-1, width)
        s0 = float(np.sum(pp[:, 0]))
        s1 = float(np.sum(pp[:, 1])) if width > 1 else 0.0
        if rparts is not None:
            rp = rparts.numpy().reshape(-1, 6)[:nrp]
            ro = rout.numpy()
            ro[0], ro[1], ro[3] = rp[:, 0].min(), rp[:, 1].max(), float(rp[:, 5].max())
            ms = max(float(rp[:, 2].max()), float(np.max(np.abs(rp[1:, 3] - rp[:-1, 4]))) if nrp > 1 else 0.0)
            ro[2] = math.inf if ro[3] else ms

        def set_res(v, conv):
            if not math.isfinite(v):
                s.status, s.res = S.KS_NONFINITE, v
                return
            s.res = v
            if conv and v <= s.tol_abs:
                s.status = S.KS_CONVERGED

        if op == S.KOP_DOT:
            out.numpy()[outoff] = s0
            return
        if op == S.KOP_NORM:
            out.numpy()[outoff] = math.sqrt(s0)
            return
        if op == S.KOP_ALPHA:
            s.pq = s0
            if s.rho == 0.0 or s0 == 0.0:
                s.status = S.KS_BREAKDOWN
            else:
                s.alpha = s.rho / s0
        elif op == S.KOP_BETA:
            s.beta = s0 / s.rho
            s.rho = s0
            s.rr = s1
            s.iteration += 1
            set_res(math.sqrt(s1), True)
        elif op in (S.KOP_REBUILD_INIT, S.KOP_REBUILD_STEP):
            s.rho, s.rr = s0, s1
            set_res(math.sqrt(s1), op == S.KOP_REBUILD_INIT)
        elif op in (S.KOP_RESID, S.KOP_RESID_INIT):
            s.rr = s1 if width > 1 else s0
            if op == S.KOP_RESID:
                s.iteration += 1
            set_res(math.sqrt(s.rr), True)
        self._put(sc, s)
        if out is not None:
            out.numpy()[outoff] = s.res
