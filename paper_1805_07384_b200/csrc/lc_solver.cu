// lc_solver.cu -- on-GPU solver harness kernels (sm_100a): 7-point constant
// coefficient stencil SpMV, fused Jacobi step, axpy / dot / norm with
// deterministic reductions.
//
// Replaces the CPU pieces the reference's solvers run per iteration
// (solvers.py:92-241: JacobiSolver, CgSolver, GmresSolver) and spmv
// (sparse.py:21-28, 150-157) for the stencil matrices of BASELINE.json's
// configs (sparse.py:184-206 generate_poisson2d; 3-D 7-point Laplacian and
// upwind convection-diffusion).  The stencil sum is accumulated in the CSR
// column order of those matrices (z-1, y-1, x-1, centre, x+1, y+1, z+1), one
// rounded multiply and add per term (no FMA, -fmad=false), so y = A x is
// bit-identical to the reference's sequential CSR accumulation.
#include "lc_kernels.cuh"
#include "../../include/lossyckpt_b200.h"

struct LcStencilDev {
    long long nx, ny, nz;
    double c, xm, xp, ym, yp, zm, zp;      // centre and neighbour coefficients
};

__device__ __forceinline__ double lc_stencil_row(const LcStencilDev &S, const double *__restrict__ x, long long k)
{
    const long long nxy = S.nx * S.ny;
    const long long iz = k / nxy, rem = k - iz * nxy, iy = rem / S.nx, ix = rem - iy * S.nx;
    double acc = 0.0;
    if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(S.zm, x[k - nxy]));
    if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(S.ym, x[k - S.nx]));
    if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(S.xm, x[k - 1]));
    acc = __dadd_rn(acc, __dmul_rn(S.c, x[k]));
    if (ix < S.nx - 1) acc = __dadd_rn(acc, __dmul_rn(S.xp, x[k + 1]));
    if (iy < S.ny - 1) acc = __dadd_rn(acc, __dmul_rn(S.yp, x[k + S.nx]));
    if (iz < S.nz - 1) acc = __dadd_rn(acc, __dmul_rn(S.zp, x[k + nxy]));
    return acc;
}

// per-block partial sums of squares / products, reduced in a fixed order
__device__ __forceinline__ void lc_block_sum(double v, double *partials)
{
    __shared__ double sw[32];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sw[w];
        partials[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(256) lc_stencil_kernel(LcStencilDev S, const double *__restrict__ x,
                                                        double *__restrict__ y, long long n)
{
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        y[k] = lc_stencil_row(S, x, k);
}

// r = b - A x, partial sums of r^2
__global__ void __launch_bounds__(256) lc_residual_kernel(LcStencilDev S, const double *__restrict__ x,
                                                         const double *__restrict__ b, double *__restrict__ r,
                                                         long long n, double *__restrict__ partials)
{
    double s = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const double v = __dsub_rn(b[k], lc_stencil_row(S, x, k));
        r[k] = v;
        s = __dadd_rn(s, __dmul_rn(v, v));
    }
    lc_block_sum(s, partials);
}

// Jacobi (solvers.py:104-110): x' = x + inv*r; r' = b - A x'; x' of the
// neighbours is recomputed from (x, r) so one launch does a whole step.
__global__ void __launch_bounds__(256) lc_jacobi_kernel(LcStencilDev S, double inv, const double *__restrict__ x,
                                                       const double *__restrict__ r, const double *__restrict__ b,
                                                       double *__restrict__ x2, double *__restrict__ r2, long long n,
                                                       double *__restrict__ partials)
{
    const long long nxy = S.nx * S.ny;
    double s = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        auto xn = [&](long long q) { return __dadd_rn(x[q], __dmul_rn(inv, r[q])); };
        const long long iz = k / nxy, rem = k - iz * nxy, iy = rem / S.nx, ix = rem - iy * S.nx;
        double acc = 0.0;
        if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(S.zm, xn(k - nxy)));
        if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(S.ym, xn(k - S.nx)));
        if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(S.xm, xn(k - 1)));
        const double xk = xn(k);
        acc = __dadd_rn(acc, __dmul_rn(S.c, xk));
        if (ix < S.nx - 1) acc = __dadd_rn(acc, __dmul_rn(S.xp, xn(k + 1)));
        if (iy < S.ny - 1) acc = __dadd_rn(acc, __dmul_rn(S.yp, xn(k + S.nx)));
        if (iz < S.nz - 1) acc = __dadd_rn(acc, __dmul_rn(S.zp, xn(k + nxy)));
        const double v = __dsub_rn(b[k], acc);
        x2[k] = xk;
        r2[k] = v;
        s = __dadd_rn(s, __dmul_rn(v, v));
    }
    lc_block_sum(s, partials);
}

__global__ void __launch_bounds__(256) lc_dot_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                                    long long n, double *__restrict__ partials)
{
    double s = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        s = __dadd_rn(s, __dmul_rn(a[k], b[k]));
    lc_block_sum(s, partials);
}

// fixed-order final sum of the block partials (one warp)
__global__ void lc_sum_kernel(const double *__restrict__ partials, int np, double *__restrict__ out)
{
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) s += partials[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
}

// y = a*x + y with a read from device memory when aptr is set (scale = sign)
__global__ void __launch_bounds__(256) lc_axpy_kernel(double a, const double *__restrict__ aptr, double scale,
                                                     const double *__restrict__ x, double *__restrict__ y, long long n)
{
    const double al = aptr ? __dmul_rn(scale, *aptr) : a;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        y[k] = __dadd_rn(y[k], __dmul_rn(al, x[k]));
}

// ---------------------------------------------------------------------------
// C ABI

struct lc_ctx;
cudaStream_t lc_stream(lc_ctx *ctx);
int lc_sm_count(lc_ctx *ctx);
void lc_count_launch(lc_ctx *ctx, int k);
int lc_fail(lc_ctx *ctx, cudaError_t e, const char *what, const char *file, int line);
void *lc_solver_scratch(lc_ctx *ctx, size_t bytes);

static LcStencilDev lc_stencil_dev(const lc_stencil *s)
{
    LcStencilDev d;
    d.nx = s->nx; d.ny = s->ny; d.nz = s->nz;
    d.c = s->c; d.xm = s->xm; d.xp = s->xp; d.ym = s->ym; d.yp = s->yp; d.zm = s->zm; d.zp = s->zp;
    return d;
}

static int lc_grid(lc_ctx *ctx, long long n)
{
    const long long g = (n + 255) / 256;
    const long long cap = 4LL * lc_sm_count(ctx);
    return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

#define LC_SOLVER_OK(x)                                                          \
    do {                                                                         \
        cudaError_t _e = (x);                                                    \
        if (_e != cudaSuccess) return lc_fail(ctx, _e, #x, __FILE__, __LINE__);  \
    } while (0)

static int lc_finish_sum(lc_ctx *ctx, double *partials, int np, double *dst_dev, double *host_out)
{
    cudaStream_t st = lc_stream(ctx);
    lc_sum_kernel<<<1, 32, 0, st>>>(partials, np, dst_dev);
    lc_count_launch(ctx, 1);
    if (host_out) {
        LC_SOLVER_OK(cudaMemcpyAsync(host_out, dst_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
        LC_SOLVER_OK(cudaStreamSynchronize(st));
    }
    LC_SOLVER_OK(cudaGetLastError());
    return 0;
}

extern "C" {

int lc_stencil_apply_f64(lc_ctx *ctx, const lc_stencil *s, const double *x, double *y)
{
    if (!ctx || !s) return 12;
    const long long n = s->nx * s->ny * s->nz;
    lc_stencil_kernel<<<lc_grid(ctx, n), 256, 0, lc_stream(ctx)>>>(lc_stencil_dev(s), x, y, n);
    lc_count_launch(ctx, 1);
    LC_SOLVER_OK(cudaGetLastError());
    return 0;
}

int lc_residual_f64(lc_ctx *ctx, const lc_stencil *s, const double *x, const double *b, double *r,
                    double *sumsq_dev, double *sumsq_host)
{
    if (!ctx || !s) return 12;
    const long long n = s->nx * s->ny * s->nz;
    const int g = lc_grid(ctx, n);
    double *partials = (double *)lc_solver_scratch(ctx, (size_t)(g + 2) * sizeof(double));
    if (!partials) return 20;
    lc_residual_kernel<<<g, 256, 0, lc_stream(ctx)>>>(lc_stencil_dev(s), x, b, r, n, partials);
    lc_count_launch(ctx, 1);
    return lc_finish_sum(ctx, partials, g, sumsq_dev ? sumsq_dev : partials + g, sumsq_host);
}

int lc_jacobi_step_f64(lc_ctx *ctx, const lc_stencil *s, double inv_diag, const double *x, const double *r,
                       const double *b, double *x_out, double *r_out, double *sumsq_dev, double *sumsq_host)
{
    if (!ctx || !s) return 12;
    const long long n = s->nx * s->ny * s->nz;
    const int g = lc_grid(ctx, n);
    double *partials = (double *)lc_solver_scratch(ctx, (size_t)(g + 2) * sizeof(double));
    if (!partials) return 20;
    lc_jacobi_kernel<<<g, 256, 0, lc_stream(ctx)>>>(lc_stencil_dev(s), inv_diag, x, r, b, x_out, r_out, n, partials);
    lc_count_launch(ctx, 1);
    return lc_finish_sum(ctx, partials, g, sumsq_dev ? sumsq_dev : partials + g, sumsq_host);
}

int lc_dot_f64(lc_ctx *ctx, const double *a, const double *b, uint64_t n, double *dot_dev, double *dot_host)
{
    if (!ctx) return 12;
    const int g = lc_grid(ctx, (long long)n);
    double *partials = (double *)lc_solver_scratch(ctx, (size_t)(g + 2) * sizeof(double));
    if (!partials) return 20;
    lc_dot_kernel<<<g, 256, 0, lc_stream(ctx)>>>(a, b, (long long)n, partials);
    lc_count_launch(ctx, 1);
    return lc_finish_sum(ctx, partials, g, dot_dev ? dot_dev : partials + g, dot_host);
}

int lc_axpy_f64(lc_ctx *ctx, double a, const double *a_dev, double a_scale, const double *x, double *y, uint64_t n)
{
    if (!ctx) return 12;
    lc_axpy_kernel<<<lc_grid(ctx, (long long)n), 256, 0, lc_stream(ctx)>>>(a, a_dev, a_scale, x, y, (long long)n);
    lc_count_launch(ctx, 1);
    LC_SOLVER_OK(cudaGetLastError());
    return 0;
}

}  // extern "C"
