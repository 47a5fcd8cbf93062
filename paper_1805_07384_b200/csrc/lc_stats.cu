// lc_stats.cu -- distortion statistics in one fused pass (sm_100a).
//
// Replaces the numpy reductions of measured_psnr (compressor.py:81-94) and
// error_identity_check (compressor.py:443-460): sum of squared errors
// (Neumaier-compensated), max |error|, value range of the original and the
// error-identity deviation max |(x - x~)_i - (pe - pe_rec)_{i-1}|, reading
// each input once.
#include "lc_kernels.cuh"

__device__ __forceinline__ void lc_neumaier(double &s, double &c, double x)
{
    const double t = s + x;
    c += fabs(s) >= fabs(x) ? (s - t) + x : (x - t) + s;
    s = t;
}

__global__ void __launch_bounds__(256) lc_stats_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                                      uint64_t n, const double *__restrict__ pe,
                                                      const double *__restrict__ pr, LcStatsPart *__restrict__ parts)
{
    double s = 0.0, c = 0.0, mx = 0.0, vmin = INFINITY, vmax = -INFINITY, dev = 0.0;
    int nf = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double x = __ldcs(a + i), y = __ldcs(b + i);
        const double d = x - y;
        lc_neumaier(s, c, d * d);
        mx = fmax(mx, fabs(d));
        vmin = fmin(vmin, x);
        vmax = fmax(vmax, x);
        nf |= !isfinite(x) | !isfinite(y);
        if (pe) dev = fmax(dev, i == 0 ? fabs(d) : fabs(d - (__ldcs(pe + i - 1) - __ldcs(pr + i - 1))));
    }
    __shared__ LcStatsPart sp[8];
    for (int o = 16; o; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, s, o), c2 = __shfl_xor_sync(0xffffffffu, c, o);
        lc_neumaier(s, c, s2);
        c += c2;
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sp[w] = LcStatsPart{s, c, mx, vmin, vmax, dev, nf, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
        LcStatsPart r = sp[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            lc_neumaier(r.sum, r.comp, sp[k].sum);
            r.comp += sp[k].comp;
            r.maxabs = fmax(r.maxabs, sp[k].maxabs);
            r.vmin = fmin(r.vmin, sp[k].vmin);
            r.vmax = fmax(r.vmax, sp[k].vmax);
            r.dev = fmax(r.dev, sp[k].dev);
            r.nonfinite |= sp[k].nonfinite;
        }
        parts[blockIdx.x] = r;
    }
}

// one thread: partials in block order (deterministic)
__global__ void lc_stats_final_kernel(const LcStatsPart *__restrict__ parts, int np, LcStatsPart *__restrict__ out)
{
    LcStatsPart r = parts[0];
    for (int k = 1; k < np; ++k) {
        lc_neumaier(r.sum, r.comp, parts[k].sum);
        r.comp += parts[k].comp;
        r.maxabs = fmax(r.maxabs, parts[k].maxabs);
        r.vmin = fmin(r.vmin, parts[k].vmin);
        r.vmax = fmax(r.vmax, parts[k].vmax);
        r.dev = fmax(r.dev, parts[k].dev);
        r.nonfinite |= parts[k].nonfinite;
    }
    *out = r;
}
