// lc_krylov.cu -- device-resident Krylov harness (sm_100a): slab-sharded
// stencil SpMV, CG / Jacobi / GMRES vector steps whose scalars never leave
// the device, deterministic chunked reductions and the value range of the
// iterate fused into the kernel that produces it.
//
// Replaces the per-iteration CPU work of the reference solvers
// (solvers.py:92-241: JacobiSolver.step, CgSolver._rebuild/step,
// GmresSolver._rebuild/_finalize_cycle/step) and spmv (sparse.py:21-28,
// 150-157) for the stencil matrices of BASELINE.json's configs.
//
// Slabs.  A rank owns global planes [z0, z0 + nzl) of an nx*ny*nz grid.  A
// vector that a stencil reads is passed as `vh`, the address of its first
// local element; vh[-plane..-1] and vh[n..n+plane) are the halo planes from
// the neighbouring ranks (only read where a neighbour exists, so one GPU
// needs no halo storage).  Rows accumulate in the reference's CSR column
// order (z-1, y-1, x-1, centre, x+1, y+1, z+1) with unfused multiply/add.
//
// Reductions.  Every dot product is a sum of per-CHUNK partials, a chunk
// being 4096 consecutive elements of the GLOBAL vector (thread t of a
// 256-thread CTA sums elements t, t+256, ... of the chunk in order; a fixed
// xor-butterfly + sequential warp fold combines the threads).  A rank's
// slab starts on a chunk boundary (the host checks nx*ny*z0 % 4096 == 0), so
// the global partial array is the concatenation of the ranks' arrays and
// lc_kr_fold_kernel sums it in one fixed order: sharded runs give the same
// bits as one GPU for any number of ranks.
//
// Scalars.  rho, alpha, beta, the residual norm, the iteration count and a
// status word live in an lc_kscalars block on the device; fold kernels
// update them, vector kernels read them.  Once the status is non-zero
// (converged, breakdown, non-finite residual) every later kernel of the
// solver returns at once, so the host may queue many iterations and read
// the status once (one host sync per batch instead of several per step).
#include "lc_kernels.cuh"
#include "../../include/lossyckpt_b200.h"

#define LC_KR_TPB 256
#define LC_KR_EPT 16
#define LC_KR_CHUNK (LC_KR_TPB * LC_KR_EPT)
#define LC_KR_FOLD_TPB 1024

static_assert(LC_KR_CHUNK == LC_KR_CHUNK_ELEMS, "chunk size must match the header");

struct LcSlabDev {
    long long nx, ny, nz, z0, nzl, plane, n;
    double c, xm, xp, ym, yp, zm, zp;
};

static LcSlabDev lc_slab_dev(const lc_slab *s)
{
    LcSlabDev d;
    d.nx = s->st.nx; d.ny = s->st.ny; d.nz = s->st.nz;
    d.z0 = s->z0; d.nzl = s->nzl;
    d.plane = d.nx * d.ny;
    d.n = d.plane * d.nzl;
    d.c = s->st.c; d.xm = s->st.xm; d.xp = s->st.xp; d.ym = s->st.ym; d.yp = s->st.yp;
    d.zm = s->st.zm; d.zp = s->st.zp;
    return d;
}

__device__ __forceinline__ double lc_kr_row(const LcSlabDev &S, const double *__restrict__ vh, long long k)
{
    const long long lz = k / S.plane, rem = k - lz * S.plane, iy = rem / S.nx, ix = rem - iy * S.nx;
    const long long iz = S.z0 + lz;
    double acc = 0.0;
    if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(S.zm, vh[k - S.plane]));
    if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(S.ym, vh[k - S.nx]));
    if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(S.xm, vh[k - 1]));
    acc = __dadd_rn(acc, __dmul_rn(S.c, vh[k]));
    if (ix < S.nx - 1) acc = __dadd_rn(acc, __dmul_rn(S.xp, vh[k + 1]));
    if (iy < S.ny - 1) acc = __dadd_rn(acc, __dmul_rn(S.yp, vh[k + S.nx]));
    if (iz < S.nz - 1) acc = __dadd_rn(acc, __dmul_rn(S.zp, vh[k + S.plane]));
    return acc;
}

// Fixed-order CTA sum of W values per thread (LC_KR_TPB threads); the result
// is valid in thread 0.  sw: W * 8 doubles of shared memory.
template <int W>
__device__ __forceinline__ void lc_kr_cta_sum(double (&v)[W], double *sw)
{
#pragma unroll
    for (int w = 0; w < W; ++w)
#pragma unroll
        for (int o = 16; o; o >>= 1) v[w] = __dadd_rn(v[w], __shfl_xor_sync(0xffffffffu, v[w], o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();                                   // sw reuse across chunks
    if (lane == 0)
#pragma unroll
        for (int w = 0; w < W; ++w) sw[w * 8 + wid] = v[w];
    __syncthreads();
    if (threadIdx.x == 0)
#pragma unroll
        for (int w = 0; w < W; ++w) {
            double s = sw[w * 8];
            for (int i = 1; i < LC_KR_TPB / 32; ++i) s = __dadd_rn(s, sw[w * 8 + i]);
            v[w] = s;
        }
}

__device__ __forceinline__ bool lc_kr_stopped(const lc_kscalars *sc) { return sc && *(volatile const int *)&sc->status; }

// Per-chunk range partial of the iterate: min, max, non-finite flag, the
// largest |x_k - x_{k-1}| inside the chunk and the chunk's first and last
// values (the step across a chunk boundary is folded by lc_kr_fold_kernel).
// The compressor's value-range record (lc_compress_ranged_f64) needs all of
// them: vmin/vmax/non-finite for the bounds and maxstep for the test that
// rules out definite escapes (no anchor pass, compressor.py:384-387).
struct LcKrRange {
    double vmin, vmax, maxstep, first, last;
    int nonfinite, pad;
};

// xv[j] = new value of element base + tid + 256 j (valid when < n).  All
// threads of the CTA call it.
__device__ __forceinline__ void lc_kr_range_chunk(const double (&xv)[LC_KR_EPT], long long base, long long n,
                                                  LcKrRange *rp, long long c)
{
    __shared__ double s_l31[LC_KR_TPB / 32][LC_KR_EPT];          // lane-31 value of each warp, per j
    __shared__ double smn[LC_KR_TPB / 32], smx[LC_KR_TPB / 32], sms[LC_KR_TPB / 32];
    __shared__ int snf[LC_KR_TPB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    __syncthreads();                                              // smem reuse across chunks
    if (lane == 31)
#pragma unroll
        for (int j = 0; j < LC_KR_EPT; ++j) s_l31[wid][j] = xv[j];
    __syncthreads();
    double mn = INFINITY, mx = -INFINITY, ms = 0.0;
    int nf = 0;
#pragma unroll
    for (int j = 0; j < LC_KR_EPT; ++j) {
        const double up = __shfl_up_sync(0xffffffffu, xv[j], 1);
        const long long k = base + tid + (long long)j * LC_KR_TPB;
        if (k < n) {
            const double v = xv[j];
            mn = fmin(mn, v); mx = fmax(mx, v); nf |= !isfinite(v);
            if (k > base) {
                const double prev = lane > 0 ? up : (wid > 0 ? s_l31[wid - 1][j] : s_l31[LC_KR_TPB / 32 - 1][j - 1]);
                ms = fmax(ms, fabs(__dsub_rn(v, prev)));
            }
            if (k == base) rp[c].first = v;
            if (k == min(base + LC_KR_CHUNK, n) - 1) rp[c].last = v;
        }
    }
    for (int o = 16; o; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (lane == 0) { smn[wid] = mn; smx[wid] = mx; sms[wid] = ms; snf[wid] = nf; }
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < LC_KR_TPB / 32; ++i) {
            mn = fmin(mn, smn[i]); mx = fmax(mx, smx[i]); ms = fmax(ms, sms[i]); nf |= snf[i];
        }
        rp[c].vmin = mn; rp[c].vmax = mx; rp[c].maxstep = ms; rp[c].nonfinite = nf;
    }
}

// ---------------------------------------------------------------------------
// kernels

// y = A vh over the slab; part[c] (optional) = sum over chunk c of vh*y
// (CG: p.q).  Skipped once sc->status is set.
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_spmv_kernel(LcSlabDev S, const double *__restrict__ vh,
                                                              double *__restrict__ y, double *__restrict__ part,
                                                              const lc_kscalars *sc)
{
    if (lc_kr_stopped(sc)) return;
    __shared__ double sw[8];
    const long long nch = (S.n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double s[1] = {0.0};
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll 4
        for (int j = 0; j < LC_KR_EPT; ++j) {
            const long long k = base + (long long)j * LC_KR_TPB;
            if (k < S.n) {
                const double v = lc_kr_row(S, vh, k);
                y[k] = v;
                s[0] = __dadd_rn(s[0], __dmul_rn(vh[k], v));
            }
        }
        if (part) {
            lc_kr_cta_sum<1>(s, sw);
            if (threadIdx.x == 0) part[c] = s[0];
        }
    }
}

// r = b - A xh; CG (z_p set): z = p = inv*r.  part[2c] = sum r*z (CG) or 0,
// part[2c+1] = sum r*r.  Runs regardless of the status (rebuilds).
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_residual_kernel(LcSlabDev S, const double *__restrict__ xh,
                                                                  const double *__restrict__ b,
                                                                  double *__restrict__ r, double inv,
                                                                  double *__restrict__ z_p, double *__restrict__ part,
                                                                  const lc_kscalars *sc_gate)
{
    if (lc_kr_stopped(sc_gate)) return;
    __shared__ double sw[16];
    const long long nch = (S.n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double s[2] = {0.0, 0.0};
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll 4
        for (int j = 0; j < LC_KR_EPT; ++j) {
            const long long k = base + (long long)j * LC_KR_TPB;
            if (k < S.n) {
                const double v = __dsub_rn(b[k], lc_kr_row(S, xh, k));
                r[k] = v;
                if (z_p) {
                    const double z = __dmul_rn(inv, v);
                    z_p[k] = z;
                    s[0] = __dadd_rn(s[0], __dmul_rn(v, z));
                }
                s[1] = __dadd_rn(s[1], __dmul_rn(v, v));
            }
        }
        lc_kr_cta_sum<2>(s, sw);
        if (threadIdx.x == 0) { part[2 * c] = s[0]; part[2 * c + 1] = s[1]; }
    }
}

// CG update (solvers.py:139-143): x += alpha p; r -= alpha q; z = inv*r;
// part[2c] = sum r*z, part[2c+1] = sum r*r; rp[c] = range of the new x.
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_cg_update_kernel(long long n, const double *__restrict__ p,
                                                                   const double *__restrict__ q,
                                                                   double *__restrict__ x, double *__restrict__ r,
                                                                   double inv, const lc_kscalars *sc,
                                                                   double *__restrict__ part, LcKrRange *rp)
{
    if (lc_kr_stopped(sc)) return;
    __shared__ double sw[16];
    const double alpha = sc->alpha;
    const long long nch = (n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double s[2] = {0.0, 0.0};
        double xv[LC_KR_EPT];
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll
        for (int j = 0; j < LC_KR_EPT; ++j) {
            const long long k = base + (long long)j * LC_KR_TPB;
            xv[j] = 0.0;
            if (k < n) {
                xv[j] = __dadd_rn(x[k], __dmul_rn(alpha, p[k]));
                x[k] = xv[j];
                const double rv = __dsub_rn(r[k], __dmul_rn(alpha, q[k]));
                r[k] = rv;
                s[0] = __dadd_rn(s[0], __dmul_rn(rv, __dmul_rn(inv, rv)));
                s[1] = __dadd_rn(s[1], __dmul_rn(rv, rv));
            }
        }
        lc_kr_cta_sum<2>(s, sw);
        if (threadIdx.x == 0) { part[2 * c] = s[0]; part[2 * c + 1] = s[1]; }
        if (rp) lc_kr_range_chunk(xv, c * LC_KR_CHUNK, n, rp, c);
    }
}

// CG direction (solvers.py:145): p = z + beta p with z = inv*r.
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_cg_dir_kernel(long long n, const double *__restrict__ r,
                                                                double *__restrict__ p, double inv,
                                                                const lc_kscalars *sc)
{
    if (lc_kr_stopped(sc)) return;
    const double beta = sc->beta;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        p[k] = __dadd_rn(__dmul_rn(inv, r[k]), __dmul_rn(beta, p[k]));
}

// Jacobi step (solvers.py:104-110): x2 = x + inv*r, r2 = b - A x2 with the
// neighbours' x2 recomputed from (x, r) (one launch per step, no halo of
// x2 needed: the halo planes of x and r are read instead).  part[c] = sum
// r2^2; rp[c] = range of x2.
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_jacobi_kernel(LcSlabDev S, double inv, const double *__restrict__ xh,
                                                                const double *__restrict__ rh,
                                                                const double *__restrict__ b,
                                                                double *__restrict__ x2, double *__restrict__ r2,
                                                                const lc_kscalars *sc, double *__restrict__ part,
                                                                LcKrRange *rp)
{
    if (lc_kr_stopped(sc)) {                            // stopped: carry the state over (the host swaps buffers)
        for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < S.n; k += (long long)gridDim.x * blockDim.x) {
            x2[k] = xh[k];
            r2[k] = rh[k];
        }
        return;
    }
    __shared__ double sw[8];
    const long long nch = (S.n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double s[1] = {0.0};
        double xv[LC_KR_EPT];
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll
        for (int j = 0; j < LC_KR_EPT; ++j) {
            const long long k = base + (long long)j * LC_KR_TPB;
            xv[j] = 0.0;
            if (k < S.n) {
                auto xn = [&](long long q) { return __dadd_rn(xh[q], __dmul_rn(inv, rh[q])); };
                const long long lz = k / S.plane, rem = k - lz * S.plane, iy = rem / S.nx, ix = rem - iy * S.nx;
                const long long iz = S.z0 + lz;
                double acc = 0.0;
                if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(S.zm, xn(k - S.plane)));
                if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(S.ym, xn(k - S.nx)));
                if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(S.xm, xn(k - 1)));
                const double xk = xn(k);
                acc = __dadd_rn(acc, __dmul_rn(S.c, xk));
                if (ix < S.nx - 1) acc = __dadd_rn(acc, __dmul_rn(S.xp, xn(k + 1)));
                if (iy < S.ny - 1) acc = __dadd_rn(acc, __dmul_rn(S.yp, xn(k + S.nx)));
                if (iz < S.nz - 1) acc = __dadd_rn(acc, __dmul_rn(S.zp, xn(k + S.plane)));
                const double v = __dsub_rn(b[k], acc);
                x2[k] = xk;
                r2[k] = v;
                s[0] = __dadd_rn(s[0], __dmul_rn(v, v));
                xv[j] = xk;
            }
        }
        lc_kr_cta_sum<1>(s, sw);
        if (threadIdx.x == 0) part[c] = s[0];
        if (rp) lc_kr_range_chunk(xv, c * LC_KR_CHUNK, S.n, rp, c);
    }
}

// part[c] = sum over chunk c of a*b (a == b: squares)
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_dot_kernel(long long n, const double *__restrict__ a,
                                                             const double *__restrict__ b, double *__restrict__ part,
                                                             const lc_kscalars *sc)
{
    if (lc_kr_stopped(sc)) return;
    __shared__ double sw[8];
    const long long nch = (n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double s[1] = {0.0};
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll 4
        for (int j = 0; j < LC_KR_EPT; ++j) {
            const long long k = base + (long long)j * LC_KR_TPB;
            if (k < n) s[0] = __dadd_rn(s[0], __dmul_rn(a[k], b[k]));
        }
        lc_kr_cta_sum<1>(s, sw);
        if (threadIdx.x == 0) part[c] = s[0];
    }
}

// y = y - (*h) x  (GMRES modified Gram-Schmidt, solvers.py:217-219)
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_subh_kernel(long long n, const double *__restrict__ x,
                                                              double *__restrict__ y, const double *__restrict__ h,
                                                              const lc_kscalars *sc)
{
    if (lc_kr_stopped(sc)) return;
    const double hv = *h;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        y[k] = __dsub_rn(y[k], __dmul_rn(hv, x[k]));
}

// y = x / (*d)  (GMRES basis normalisation, solvers.py:184, 237)
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_div_kernel(long long n, const double *__restrict__ x,
                                                             double *__restrict__ y, const double *__restrict__ d,
                                                             const lc_kscalars *sc)
{
    if (lc_kr_stopped(sc)) return;
    const double dv = *d;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        y[k] = __ddiv_rn(x[k], dv);
}

// GMRES solution update (solvers.py:196): x = x_base + sum_i y_i v_i, the sum
// formed in basis order (t = y_0 v_0, t += y_i v_i); rp[c] = range of x.
__global__ void __launch_bounds__(LC_KR_TPB) lc_kr_combine_kernel(long long n, int j, const double *__restrict__ basis,
                                                                 long long ld, const double *__restrict__ yv,
                                                                 const double *__restrict__ xbase,
                                                                 double *__restrict__ x, LcKrRange *rp)
{
    const long long nch = (n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
        double xv[LC_KR_EPT];
        const long long base = c * LC_KR_CHUNK + threadIdx.x;
#pragma unroll
        for (int jj = 0; jj < LC_KR_EPT; ++jj) {
            const long long k = base + (long long)jj * LC_KR_TPB;
            xv[jj] = 0.0;
            if (k < n) {
                double t = j > 0 ? __dmul_rn(yv[0], basis[k]) : 0.0;
                for (int i = 1; i < j; ++i) t = __dadd_rn(t, __dmul_rn(yv[i], basis[(long long)i * ld + k]));
                xv[jj] = j > 0 ? __dadd_rn(xbase[k], t) : xbase[k];
                x[k] = xv[jj];
            }
        }
        if (rp) lc_kr_range_chunk(xv, c * LC_KR_CHUNK, n, rp, c);
    }
}

__device__ __forceinline__ void lc_kr_set_residual(lc_kscalars *sc, double v, bool conv_test)
{
    if (!isfinite(v)) { sc->status = LC_KS_NONFINITE; sc->res = v; return; }
    sc->res = v;
    if (conv_test && v <= sc->tol_abs) sc->status = LC_KS_CONVERGED;
}

// Fold the global partial array part[nch][W] in one fixed order and apply op
// (LC_KOP_*) to the scalars; rp/nrp (optional): fold the range partials of
// the local iterate into *rout (maxstep = vmax - vmin, an upper bound of
// every |x_i - x_{i-1}|).  One CTA.
__global__ void __launch_bounds__(LC_KR_FOLD_TPB) lc_kr_fold_kernel(const double *__restrict__ part, int W,
                                                                   long long nch, int op, lc_kscalars *sc,
                                                                   double *__restrict__ out,
                                                                   const LcKrRange *__restrict__ rp, long long nrp,
                                                                   LcRangePart *rout)
{
    __shared__ double sw[2][32];
    __shared__ int s_stop;
    // DOT / NORM / *_INIT run unconditionally; the in-iteration ops stop with the solver
    if (threadIdx.x == 0)
        s_stop = (op == LC_KOP_ALPHA || op == LC_KOP_BETA || op == LC_KOP_REBUILD_STEP || op == LC_KOP_RESID) &&
                 sc->status != LC_KS_RUNNING;
    __syncthreads();
    if (s_stop) return;
    double s0 = 0.0, s1 = 0.0;
    for (long long c = threadIdx.x; c < nch; c += LC_KR_FOLD_TPB) {
        s0 = __dadd_rn(s0, part[c * W]);
        if (W > 1) s1 = __dadd_rn(s1, part[c * W + 1]);
    }
    for (int o = 16; o; o >>= 1) {
        s0 = __dadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
        s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { sw[0][wid] = s0; sw[1][wid] = s1; }
    // range of the iterate (order-free: min/max)
    double mn = INFINITY, mx = -INFINITY, ms = 0.0;
    int nf = 0;
    if (rp)
        for (long long c = threadIdx.x; c < nrp; c += LC_KR_FOLD_TPB) {
            mn = fmin(mn, rp[c].vmin); mx = fmax(mx, rp[c].vmax); nf |= rp[c].nonfinite;
            ms = fmax(ms, rp[c].maxstep);
            if (c > 0) ms = fmax(ms, fabs(__dsub_rn(rp[c].first, rp[c - 1].last)));   // across the boundary
        }
    __syncthreads();
    if (wid == 0) {
        s0 = sw[0][lane];
        s1 = sw[1][lane];
        for (int o = 16; o; o >>= 1) {
            s0 = __dadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
            s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        }
    }
    if (rp) {
        __shared__ double smn[32], smx[32], sms[32];
        __shared__ int snf[32];
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
            nf |= __shfl_xor_sync(0xffffffffu, nf, o);
        }
        if (lane == 0) { smn[wid] = mn; smx[wid] = mx; sms[wid] = ms; snf[wid] = nf; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < LC_KR_FOLD_TPB / 32; ++i) {
                mn = fmin(mn, smn[i]); mx = fmax(mx, smx[i]); ms = fmax(ms, sms[i]); nf |= snf[i];
            }
            rout->vmin = mn; rout->vmax = mx; rout->nonfinite = nf;
            rout->maxstep = nf ? INFINITY : ms;
        }
    }
    if (threadIdx.x != 0) return;
    switch (op) {
    case LC_KOP_DOT:                                     // out = sum
        *out = s0;
        break;
    case LC_KOP_NORM:                                    // out = sqrt(sum)
        *out = __dsqrt_rn(s0);
        break;
    case LC_KOP_ALPHA:                                   // CG: pq, alpha = rho / pq
        sc->pq = s0;
        if (sc->rho == 0.0 || s0 == 0.0) { sc->status = LC_KS_BREAKDOWN; break; }
        sc->alpha = __ddiv_rn(sc->rho, s0);
        break;
    case LC_KOP_BETA: {                                  // CG: rho_new, beta, residual
        const double rho_new = s0;
        sc->beta = __ddiv_rn(rho_new, sc->rho);
        sc->rho = rho_new;
        sc->rr = s1;
        sc->iteration += 1;
        lc_kr_set_residual(sc, __dsqrt_rn(s1), true);
        break;
    }
    case LC_KOP_REBUILD_INIT:                            // CG rebuild (fresh state): rho, residual, converged
    case LC_KOP_REBUILD_STEP:                            // restart inside a step: no convergence test
        sc->rho = s0;
        sc->rr = s1;
        lc_kr_set_residual(sc, __dsqrt_rn(s1), op == LC_KOP_REBUILD_INIT);
        break;
    case LC_KOP_RESID:                                   // Jacobi: residual of the step just taken
        sc->rr = W > 1 ? s1 : s0;                        // (width 2: lc_kr_residual_f64's r.r column)
        sc->iteration += 1;
        lc_kr_set_residual(sc, __dsqrt_rn(sc->rr), true);
        break;
    case LC_KOP_RESID_INIT:                              // residual of a (re)built state
        sc->rr = W > 1 ? s1 : s0;
        lc_kr_set_residual(sc, __dsqrt_rn(sc->rr), true);
        break;
    default:
        break;
    }
    if (out && op != LC_KOP_DOT && op != LC_KOP_NORM) *out = sc->res;
}

// ---------------------------------------------------------------------------
// C ABI

struct lc_ctx;
cudaStream_t lc_stream(lc_ctx *ctx);
int lc_sm_count(lc_ctx *ctx);
void lc_count_launch(lc_ctx *ctx, int k);
int lc_fail(lc_ctx *ctx, cudaError_t e, const char *what, const char *file, int line);

#define LC_KR_OK(x)                                                              \
    do {                                                                         \
        cudaError_t _e = (x);                                                    \
        if (_e != cudaSuccess) return lc_fail(ctx, _e, #x, __FILE__, __LINE__);  \
    } while (0)

static int lc_kr_grid_chunks(lc_ctx *ctx, long long n)
{
    const long long nch = (n + LC_KR_CHUNK - 1) / LC_KR_CHUNK;
    const long long cap = 8LL * lc_sm_count(ctx);          // 8 resident 256-thread CTAs per SM
    return (int)(nch < cap ? (nch > 0 ? nch : 1) : cap);
}

static int lc_kr_grid_elems(lc_ctx *ctx, long long n)
{
    const long long g = (n + LC_KR_TPB - 1) / LC_KR_TPB;
    const long long cap = 8LL * lc_sm_count(ctx);
    return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

static int lc_kr_done(lc_ctx *ctx)
{
    lc_count_launch(ctx, 1);
    LC_KR_OK(cudaGetLastError());
    return 0;
}

static bool lc_slab_ok(const lc_slab *s)
{
    return s && s->st.nx > 0 && s->st.ny > 0 && s->st.nz > 0 && s->z0 >= 0 && s->nzl > 0 &&
           s->z0 + s->nzl <= s->st.nz;
}

extern "C" {

int lc_kr_spmv_f64(lc_ctx *ctx, const lc_slab *s, const double *vh, double *y, double *part,
                   const lc_kscalars *sc)
{
    if (!ctx || !lc_slab_ok(s)) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    const LcSlabDev S = lc_slab_dev(s);
    lc_kr_spmv_kernel<<<lc_kr_grid_chunks(ctx, S.n), LC_KR_TPB, 0, lc_stream(ctx)>>>(S, vh, y, part, sc);
    return lc_kr_done(ctx);
}

int lc_kr_residual_f64(lc_ctx *ctx, const lc_slab *s, const double *xh, const double *b, double *r,
                       double inv_diag, double *z_p, double *part, const lc_kscalars *sc_gate)
{
    if (!ctx || !lc_slab_ok(s) || !part) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    const LcSlabDev S = lc_slab_dev(s);
    lc_kr_residual_kernel<<<lc_kr_grid_chunks(ctx, S.n), LC_KR_TPB, 0, lc_stream(ctx)>>>(S, xh, b, r, inv_diag, z_p,
                                                                                      part, sc_gate);
    return lc_kr_done(ctx);
}

int lc_kr_cg_update_f64(lc_ctx *ctx, uint64_t n, const double *p, const double *q, double *x, double *r,
                        double inv_diag, const lc_kscalars *sc, double *part, void *range_parts)
{
    if (!ctx || !sc || !part) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_cg_update_kernel<<<lc_kr_grid_chunks(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>(
        (long long)n, p, q, x, r, inv_diag, sc, part, (LcKrRange *)range_parts);
    return lc_kr_done(ctx);
}

int lc_kr_cg_dir_f64(lc_ctx *ctx, uint64_t n, const double *r, double *p, double inv_diag, const lc_kscalars *sc)
{
    if (!ctx || !sc) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_cg_dir_kernel<<<lc_kr_grid_elems(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>((long long)n, r, p,
                                                                                            inv_diag, sc);
    return lc_kr_done(ctx);
}

int lc_kr_jacobi_f64(lc_ctx *ctx, const lc_slab *s, double inv_diag, const double *xh, const double *rh,
                     const double *b, double *x2, double *r2, const lc_kscalars *sc, double *part,
                     void *range_parts)
{
    if (!ctx || !lc_slab_ok(s) || !part) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    const LcSlabDev S = lc_slab_dev(s);
    lc_kr_jacobi_kernel<<<lc_kr_grid_chunks(ctx, S.n), LC_KR_TPB, 0, lc_stream(ctx)>>>(
        S, inv_diag, xh, rh, b, x2, r2, sc, part, (LcKrRange *)range_parts);
    return lc_kr_done(ctx);
}

int lc_kr_dot_f64(lc_ctx *ctx, uint64_t n, const double *a, const double *b, double *part, const lc_kscalars *sc)
{
    if (!ctx || !part) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_dot_kernel<<<lc_kr_grid_chunks(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>((long long)n, a, b,
                                                                                          part, sc);
    return lc_kr_done(ctx);
}

int lc_kr_subh_f64(lc_ctx *ctx, uint64_t n, const double *x, double *y, const double *h_dev, const lc_kscalars *sc)
{
    if (!ctx || !h_dev) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_subh_kernel<<<lc_kr_grid_elems(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>((long long)n, x, y,
                                                                                          h_dev, sc);
    return lc_kr_done(ctx);
}

int lc_kr_div_f64(lc_ctx *ctx, uint64_t n, const double *x, double *y, const double *d_dev, const lc_kscalars *sc)
{
    if (!ctx || !d_dev) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_div_kernel<<<lc_kr_grid_elems(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>((long long)n, x, y,
                                                                                         d_dev, sc);
    return lc_kr_done(ctx);
}

int lc_kr_combine_f64(lc_ctx *ctx, uint64_t n, int j, const double *basis, uint64_t ld, const double *y_dev,
                      const double *xbase, double *x, void *range_parts)
{
    if (!ctx || j < 0 || (j > 0 && (!basis || !y_dev))) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_combine_kernel<<<lc_kr_grid_chunks(ctx, (long long)n), LC_KR_TPB, 0, lc_stream(ctx)>>>(
        (long long)n, j, basis, (long long)ld, y_dev, xbase, x, (LcKrRange *)range_parts);
    return lc_kr_done(ctx);
}

int lc_kr_fold_f64(lc_ctx *ctx, const double *part, int width, uint64_t nchunks, int op, lc_kscalars *sc,
                   double *out_dev, const void *range_parts, uint64_t n_range_parts, void *range_out)
{
    if (!ctx || !part || (width != 1 && width != 2)) return 12;
    if (op != LC_KOP_DOT && op != LC_KOP_NORM && !sc) return 12;
    if ((op == LC_KOP_DOT || op == LC_KOP_NORM) && !out_dev) return 12;
    LcDeviceGuard guard(lc_ctx_device(ctx));
    lc_kr_fold_kernel<<<1, LC_KR_FOLD_TPB, 0, lc_stream(ctx)>>>(part, width, (long long)nchunks, op, sc, out_dev,
                                                               (const LcKrRange *)range_parts,
                                                               (long long)n_range_parts, (LcRangePart *)range_out);
    return lc_kr_done(ctx);
}

}  // extern "C"
