// lc_quant.cu -- value range + fused exact-chain quantizer (sm_100a).
//
// Replaces compressor.py:384-386 (isfinite/min/max) and the sequential
// _compress_kernel (compressor.py:319-355) + np.bincount (compressor.py:411).
//
// lc_quant_kernel processes tiles of 256 chunks x 32 elements with a
// persistent grid and two decoupled look-backs per tile:
//   phase 0  definite-escape positions (max scan): anchors the guesses
//   phase A  guess chain per chunk -> offset map (lc_chain.cuh)
//            block scan + look-back of the maps -> exact start of each chunk
//   phase B  exact reference chain from that start: codes, histogram,
//            optional traces; each chunk checks its end against the next
//            chunk's predicted start (first failure -> host relaunch).
#include <cub/block/block_scan.cuh>
#include "lc_kernels.cuh"

// kernel entry: take the device-resolved bounds (written by
// lc_quant_setup_kernel earlier in the same stream; every CTA reads the
// context's own LcQuantDyn through the read-only path into registers, so
// concurrent calls on other streams and contexts never share them);
// false = nothing to do
__device__ __forceinline__ bool lc_quant_dyn(LcQuantParams &P)
{
    if (!P.dyn) return true;
    const LcQuantDyn *d = P.dyn;
    if (__ldg(&d->skip)) return false;
    P.Q.delta = __ldg(&d->Q.delta);
    P.Q.eb = __ldg(&d->Q.eb);
    P.Q.max_m = __ldg(&d->Q.max_m);
    P.Q.max_m1 = __ldg(&d->Q.max_m1);
    P.Q.inv = __ldg(&d->Q.inv);
    P.Q.cert = __ldg(&d->Q.cert);
    P.esc_thresh = __ldg(&d->esc_thresh);
    P.use_anchors = __ldg(&d->use_anchors);
    return true;
}


// ---------------------------------------------------------------------------
// range: min, max, non-finite flag


__global__ void __launch_bounds__(256) lc_range_kernel(const double *__restrict__ x, uint64_t n,
                                                      LcRangePart *__restrict__ parts, unsigned *__restrict__ done)
{
    // min, max, non-finite flag and max |x_i - x_{i-1}| (decides whether definite
    // escapes are possible, lc_compress_f64).  Each lane owns 8 consecutive
    // elements per group (four 16-byte loads, two groups in flight), so a warp
    // covers 256 contiguous elements; the predecessor of a lane's first element
    // is the previous lane's last one (lane 0 loads it).  An 8-byte aligned x
    // starts the groups at x + 1 (x[0] is folded in by thread 0).
    double mn = INFINITY, mx = -INFINITY, ms = 0.0;
    int nf = 0;
    const int lane = threadIdx.x & 31;
    const uint64_t off = (reinterpret_cast<uintptr_t>(x) & 15) ? 1 : 0;
    const double *base = x + off;
    const uint64_t nb = n > off ? n - off : 0;
    const uint64_t ngroups = nb / 8;                      // full 8-element groups
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    const double2 *x2 = reinterpret_cast<const double2 *>(base);
    auto group = [&](uint64_t g, const double (&v)[8]) {
        double prev = __shfl_up_sync(0xffffffffu, v[7], 1);
        if (lane == 0) prev = g > 0 ? base[8 * g - 1] : (off ? x[0] : v[0]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double a = v[k];
            nf |= !isfinite(a);
            mn = fmin(mn, a);
            mx = fmax(mx, a);
            ms = fmax(ms, fabs(__dsub_rn(a, k ? v[k - 1] : prev)));
        }
    };
    // warp-uniform trip counts: the warp's first group decides
    for (uint64_t wg = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wg < ngroups; wg += 2 * gstride) {
        const uint64_t g0 = wg + lane, g1 = wg + gstride + lane;
        double v0[8], v1[8];
        const bool ok0 = g0 < ngroups, ok1 = g1 < ngroups;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 a = ok0 ? __ldcs(x2 + 4 * g0 + k) : make_double2(0.0, 0.0);
            const double2 c = ok1 ? __ldcs(x2 + 4 * g1 + k) : make_double2(0.0, 0.0);
            v0[2 * k] = a.x; v0[2 * k + 1] = a.y;
            v1[2 * k] = c.x; v1[2 * k + 1] = c.y;
        }
        // lanes past the end repeat the last valid element of the warp's range
        const unsigned m0 = __ballot_sync(0xffffffffu, ok0), m1 = __ballot_sync(0xffffffffu, ok1);
        if (m0) {
            if (!ok0) {
                const double last = base[8 * (wg + (31 - __clz(m0))) + 7];
#pragma unroll
                for (int k = 0; k < 8; ++k) v0[k] = last;
            }
            group(wg, v0);
        }
        if (m1) {
            if (!ok1) {
                const double last = base[8 * (wg + gstride + (31 - __clz(m1))) + 7];
#pragma unroll
                for (int k = 0; k < 8; ++k) v1[k] = last;
            }
            group(wg + gstride, v1);
        }
    }
    // x[0] when skipped for alignment, and the tail (< 8 elements): thread 0
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (off) { const double a = x[0]; nf |= !isfinite(a); mn = fmin(mn, a); mx = fmax(mx, a); }
        for (uint64_t i = off + ngroups * 8; i < n; ++i) {
            const double a = x[i];
            nf |= !isfinite(a);
            mn = fmin(mn, a);
            mx = fmax(mx, a);
            if (i > 0) ms = fmax(ms, fabs(__dsub_rn(a, x[i - 1])));
        }
    }
    for (int o = 16; o; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    __shared__ double smn[8], smx[8], sms[8];
    __shared__ int snf[8];
    const int w = threadIdx.x >> 5;
    if (lane == 0) { smn[w] = mn; smx[w] = mx; sms[w] = ms; snf[w] = nf; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            mn = fmin(mn, smn[k]); mx = fmax(mx, smx[k]); ms = fmax(ms, sms[k]); nf |= snf[k];
        }
        parts[blockIdx.x].vmin = mn;
        parts[blockIdx.x].vmax = mx;
        parts[blockIdx.x].maxstep = ms;
        parts[blockIdx.x].nonfinite = nf;
    }
    // the last block to finish folds every block's part into parts[gridDim.x]
    // (and re-arms the counter for the next call)
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    __threadfence();
    mn = INFINITY; mx = -INFINITY; ms = 0.0; nf = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) {
        mn = fmin(mn, __ldcg(&parts[i].vmin)); mx = fmax(mx, __ldcg(&parts[i].vmax));
        ms = fmax(ms, __ldcg(&parts[i].maxstep)); nf |= __ldcg(&parts[i].nonfinite);
    }
    for (int o = 16; o; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (threadIdx.x == 0) {
        LcRangePart *out = parts + gridDim.x;
        out->vmin = mn; out->vmax = mx; out->maxstep = ms; out->nonfinite = nf;
        *done = 0u;
    }
}

// Quantizer setup on the device from the range pass (same IEEE operations as
// the host path: compressor.py resolve_bounds eb_abs = eb_rel * vr, then the
// lc_compress_f64 derivations), so relative-mode compression needs no host
// round trip before the quantizer.
__global__ void lc_quant_setup_kernel(const LcRangePart *__restrict__ r, const double *__restrict__ x, uint64_t n,
                                      int eb_relative, double eb_param, uint32_t nbh, LcQuantDyn *d)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double vmin = r->vmin, vmax = r->vmax;
    double vr = __dsub_rn(vmax, vmin);
    if (vr == 0.0) vr = 0.0;
    const double eb = eb_relative ? __dmul_rn(eb_param, vr) : eb_param;
    int st = 0;
    if (r->nonfinite) st = 10;
    else if (vr == 0.0 || n < 2) st = 15;
    else if (!isfinite(__dmul_rn(2.0, eb))) st = 11;
    else if (!(eb > 0.0)) st = 12;
    LcQuantDyn o;
    o.vmin = vmin; o.vmax = vmax; o.value_range = vr; o.eb_abs = eb; o.first_value = x[0];
    o.nonfinite = r->nonfinite;
    o.status = st;
    o.skip = st != 0;
    o.Q.delta = __dmul_rn(2.0, eb);
    o.Q.eb = eb;
    o.Q.max_m = (double)(nbh - 1);
    o.Q.max_m1 = __dadd_rn(o.Q.max_m, 1.0);
    o.Q.inv = __ddiv_rn(1.0, o.Q.delta);
    int e2;
    frexp(__dadd_rn(o.Q.max_m, 2.0), &e2);
    o.Q.cert = __dsub_rn(0.5, ldexp(1.0, e2 - 50));
    o.esc_thresh = __dmul_rn(__dmul_rn((double)nbh, o.Q.delta), 1.0 + 0x1p-40);
    const double ms = r->maxstep;
    o.use_anchors = (__dsub_rn(__dmul_rn(ms, 1.0 - 0x1p-50), __dmul_rn(eb, 1.0 + 0x1p-50)) >= o.esc_thresh) ||
                    !isfinite(ms);
    // every chain value r satisfies |r| <= max|x| + eb (kept: |x - r| <= eb, escaped: r = x)
    o.rmax = __dmul_rn(__dadd_rn(fmax(fabs(vmin), fabs(vmax)), eb), 1.0 + 0x1p-50);
    *d = o;
}

// ---------------------------------------------------------------------------
// fused quantizer


// Definite escape at element i: |pe*| >= |x_i - x_{i-1}| - eb exceeds the
// quantizer range whatever the reconstruction r*_{i-1} is (|x - r*| <= eb).
__device__ __forceinline__ bool lc_definite_escape(double xi, double xprev, const LcQuantParams &P)
{
    const double d = fabs(LC_SUB(xi, xprev));
    return LC_SUB(LC_MUL(d, 1.0 - 0x1p-50), LC_MUL(P.Q.eb, 1.0 + 0x1p-50)) >= P.esc_thresh;
}

// ---------------------------------------------------------------------------
// Anchor pre-pass (only when definite escapes are possible): the last
// definite escape of every tile and their running max (lc_quantf_kernel reads
// anc_in[t]).

__global__ void __launch_bounds__(LC_TPB) lc_anchor_tiles_kernel(LcQuantParams P)
{
    if (!lc_quant_dyn(P) || !P.use_anchors) return;
    // last definite escape position of every warp tile (escapes certain from the data)
    const int lane = threadIdx.x & 31;
    const long long nel = (long long)P.n - 1;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < P.ntiles; w += nwarps) {
        const long long pbeg = (P.first_chunk + w * 32) * LC_L;
        long long last = -1;
        for (int k = 0; k < 32; ++k) {
            const long long pos = pbeg + 1 + k * 32 + lane;
            if (pos <= nel && lc_definite_escape(P.x[pos], P.x[pos - 1], P)) last = max(last, pos);
        }
        for (int o = 16; o; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        if (lane == 0) P.tile_last_esc[w] = last;
    }
}

__global__ void __launch_bounds__(1024) lc_anchor_scan_kernel(const long long *__restrict__ last,
                                                             long long *__restrict__ incoming, long long ntiles,
                                                             long long launch_pos, const LcQuantDyn *dyn)
{
    if (dyn && (dyn->skip || !dyn->use_anchors)) return;
    typedef cub::BlockScan<long long, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = launch_pos;
    __syncthreads();
    struct MaxOp { __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; } };
    for (long long b = 0; b < ntiles; b += 1024) {
        const long long i = b + threadIdx.x;
        const long long v = i < ntiles ? last[i] : -1;
        long long ex, agg;
        Scan(tmp).ExclusiveScan(v, ex, -1LL, MaxOp(), agg);
        const long long c = carry;
        if (i < ntiles) incoming[i] = max(c, ex);
        __syncthreads();
        if (threadIdx.x == 0) carry = max(c, agg);
        __syncthreads();
    }
}

// Offsets at every tile start: D_0 = 0, D_{t+1} = agg_t(D_t).  G co-resident
// CTAs of 1024 threads (G <= SM count); thread i composes `per` consecutive tile
// maps, a block scan gives each thread's in-group exclusive map and the group
// aggregate, which is published (release flag).  Thread 0 folds the aggregates
// of all earlier groups (acquire; they never wait on later groups) into the
// offset at the group start; every thread then evaluates its tiles.
// D0p (optional): the offset at the first tile's start (resume after a failed
// prediction); 0 at a launch anchor.  A NaN offset means no resume: exit.
__global__ void __launch_bounds__(1024) lc_map_scan_kernel(const OffMap *__restrict__ agg, double *__restrict__ tileD,
                                                          long long ntiles, long long per, OffMap *gagg, int *gflag,
                                                          const double *D0p)
{
    const double D0 = D0p ? *D0p : 0.0;
    if (D0 != D0) return;
    __shared__ OffMap wsum[32];
    __shared__ double s_D;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, g = blockIdx.x;
    const long long b0 = min(ntiles, ((long long)g * 1024 + tid) * per), b1 = min(ntiles, b0 + per);
    OffMap run = lc_map_neutral();
    if (per == 1) {                                  // the usual case: no per-thread composition at all
        if (b0 < b1) run = agg[b0];
    } else {
        for (long long t = b0; t < b1; ++t) run = lc_map_compose(agg[t], run);
        __syncwarp();
    }
    OffMap inc = run;
    lc_warp_scan_maps(inc);                          // prefix sum when every map is a translation
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    lc_scan_warp_maps(wsum, 32);
    __syncthreads();
    // exclusive maps: shuffle first (the warp is converged after the scan), compose per lane
    // afterwards -- no shuffle may follow a per-lane composition (see lc_warp_scan_maps)
    OffMap exc = lc_shfl_up_map(inc, 1);
    if (lane == 0) exc = lc_map_neutral();
    if (wid > 0) {
        exc = lc_map_compose(exc, wsum[wid - 1]);
        inc = lc_map_compose(inc, wsum[wid - 1]);
    }
    if (wid == 0) {
        // publish this group's aggregate, then fold the aggregates of all earlier
        // groups 32 at a time (parallel acquire loads, shuffle-tree composition)
        if (lane == 0) {
            gagg[g] = wsum[31];
            __threadfence();
            st_release(gflag + g, 1);
        }
        OffMap acc = lc_map_neutral();
        for (int base = 0; base < g; base += 32) {
            const int j = base + lane;
            OffMap v = lc_map_neutral();
            if (j < g) {
                while (ld_acquire(gflag + j) != 1) { }
                const OffMap *q = gagg + j;         // L2 reads (written by another CTA)
                v.kind = __ldcg(&q->kind); v.v = __ldcg(&q->v); v.B = __ldcg(&q->B); v.t0 = __ldcg(&q->t0);
                v.t1 = __ldcg(&q->t1); v.y = __ldcg(&q->y); v.og = __ldcg(&q->og);
            }
            __syncwarp();
            lc_warp_scan_maps(v);                    // lane-uniform; lane 31 holds the 32 groups' composition
            acc = lc_map_compose(lc_shfl_idx_map(v, 31), acc);   // the same operands in every lane
        }
        if (lane == 0) s_D = lc_map_eval(acc, D0);
    }
    __syncthreads();
    double D = lc_map_eval(exc, s_D);
    for (long long t = b0; t < b1; ++t) {
        tileD[t] = D;
        D = lc_map_eval(agg[t], D);
    }
    if (b0 < b1 && b1 == ntiles) tileD[ntiles] = D;
}

int lc_launch_map_scan(const OffMap *agg, double *tileD, long long ntiles, void *scratch, int sm_count,
                       cudaStream_t st, const double *D0p)
{
    if (ntiles <= 0) return 0;
    long long G = (ntiles + 1023) / 1024;
    if (G > sm_count) G = sm_count;
    if (G > LC_MAPSCAN_MAXG) G = LC_MAPSCAN_MAXG;
    if (G < 1) G = 1;
    const long long per = (ntiles + 1024 * G - 1) / (1024 * G);
    OffMap *gagg = (OffMap *)scratch;
    int *gflag = (int *)(gagg + LC_MAPSCAN_MAXG);
    cudaError_t e = cudaMemsetAsync(gflag, 0, G * sizeof(int), st);
    if (e != cudaSuccess) return (int)e;
    lc_map_scan_kernel<<<(int)G, 1024, 0, st>>>(agg, tileD, ntiles, per, gagg, gflag, D0p);
    return (int)cudaGetLastError();
}

// Sequential exact chain from chunk `first_chunk` (fallback for inputs whose
// chunk predictions keep failing).  One thread; correct for every input.
template <typename CodeT>
__global__ void lc_quant_serial_kernel(LcQuantParams P, CodeT *__restrict__ codes)
{
    if (!lc_quant_dyn(P)) return;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double r = P.first_chunk == 0 ? P.x[0] : P.anchor_val;   // a launch from the start is anchored at x[0]
    for (uint64_t i = (uint64_t)P.first_chunk * LC_L + 1; i < P.n; ++i) {
        uint32_t code; int esc; double inc, pe;
        if (P.sync_start && ((i - 1) & (LC_SYNC_K - 1)) == 0) P.sync_start[(i - 1) / LC_SYNC_K] = r;
        const double rn = lc_step(P.Q, P.x[i], r, &code, &esc, &inc, &pe);
        codes[i - 1] = (CodeT)code;
        if (P.pe) { P.pe[i - 1] = pe; P.pe_rec[i - 1] = LC_SUB(rn, r); }
        r = rn;
    }
}

// v3 sync starts: the exact chain value at the start of every warp tile of this
// launch (= every LC_SYNC_K-th element; launches start on warp tiles), from
// pass A's tile guess and the map scan's exact offset -- after pass B every
// predicted tile start is the reference's value.
__global__ void lc_sync_starts_kernel(LcQuantParams P)
{
    if (!lc_quant_dyn(P) || !P.sync_start) return;
    const long long k0 = P.first_chunk / 32;
    for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < P.ntiles; w += (long long)gridDim.x * blockDim.x)
        if ((unsigned long long)(k0 + w) < P.nsync) P.sync_start[k0 + w] = lc_apply_offset(P.tile_g0[w], P.tile_D[w]);
}

// Histogram recount from final codes (used after relaunches).
template <typename CodeT>
__global__ void __launch_bounds__(256) lc_hist_kernel(const CodeT *__restrict__ codes, uint64_t m,
                                                     uint32_t *__restrict__ hist, uint32_t nbins)
{
    __shared__ uint32_t hs[LC_HBINS];
    for (int i = threadIdx.x; i < LC_HBINS; i += blockDim.x) hs[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint32_t code = codes[i];
        if (code < LC_HBINS) atomicAdd(&hs[code], 1u);
        else atomicAdd(&hist[code], 1u);
    }
    __syncthreads();
    const uint32_t lim = nbins < LC_HBINS ? nbins : LC_HBINS;
    for (uint32_t i = threadIdx.x; i < lim; i += blockDim.x)
        if (hs[i]) atomicAdd(&hist[i], hs[i]);
}

// Wide alphabets (np.bincount, compressor.py:411, for codes >= lo): pass A counts codes
// below `lo` (= its shared-memory histogram) itself and only counts how many were
// larger (*nbig); this pass streams over the final codes and counts the codes in
// [lo, lo + LC_HW_BINS) with shared-memory atomics (64 KB per CTA) and the rest with
// global ones.  Without it every such code was a global atomic on a few thousand
// addresses (config 5: 12k symbols, 134M codes, 3.4 ms).  Exits at once when no code
// was large, or when a chunk prediction failed (the quantizer is resumed first).
template <typename CodeT>
__global__ void __launch_bounds__(512) lc_histw_kernel(const CodeT *__restrict__ codes, uint64_t m,
                                                      uint32_t *__restrict__ hist, uint32_t nbins, uint32_t lo,
                                                      const unsigned long long *__restrict__ nbig,
                                                      const unsigned long long *__restrict__ pending,
                                                      const LcQuantDyn *dyn)
{
    if (dyn && dyn->skip) return;
    if (*nbig == 0 || (pending && *pending != ~0ULL)) return;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    uint32_t *hs = reinterpret_cast<uint32_t *>(lc_dyn_smem);
    for (uint32_t i = threadIdx.x; i < LC_HW_BINS; i += blockDim.x) hs[i] = 0;
    __syncthreads();
    constexpr int V = 16 / sizeof(CodeT);
    const uint64_t nv = m / V;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint4 *c4 = reinterpret_cast<const uint4 *>(codes);
    auto add = [&](uint32_t code) {
        const uint32_t r = code - lo;
        if (code >= lo) {
            if (r < LC_HW_BINS) atomicAdd(&hs[r], 1u);
            else atomicAdd(&hist[code], 1u);
        }
    };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 q = __ldcs(c4 + i);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (sizeof(CodeT) == 2) { add(w[k] & 0xffffu); add(w[k] >> 16); }
            else add(w[k]);
        }
    }
    if (blockIdx.x == 0)
        for (uint64_t i = nv * V + threadIdx.x; i < m; i += blockDim.x) add((uint32_t)codes[i]);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < LC_HW_BINS; i += blockDim.x)
        if (hs[i] && lo + i < nbins) atomicAdd(&hist[lo + i], hs[i]);
}
template __global__ void lc_histw_kernel<uint16_t>(const uint16_t *, uint64_t, uint32_t *, uint32_t, uint32_t,
                                                   const unsigned long long *, const unsigned long long *,
                                                   const LcQuantDyn *);
template __global__ void lc_histw_kernel<uint32_t>(const uint32_t *, uint64_t, uint32_t *, uint32_t, uint32_t,
                                                   const unsigned long long *, const unsigned long long *,
                                                   const LcQuantDyn *);

// Histogram of u16 codes (np.bincount, compressor.py:411) as its own streaming
// pass: 16-byte loads, codes 1..16 (the small |m| of smooth data) in packed
// per-thread byte counters flushed every 128 codes into 16 register totals,
// every other code by shared/global atomics; warp sums by redux.sync, one
// atomic per lane and code.  m codes, hist pre-zeroed.
__global__ void __launch_bounds__(256) lc_hist16_kernel(const uint16_t *__restrict__ codes, uint64_t m,
                                                      uint32_t *__restrict__ hist, uint32_t nbins,
                                                      const LcQuantDyn *dyn)
{
    if (dyn && dyn->skip) return;
    __shared__ uint32_t hs[LC_HBINS];
    for (int i = threadIdx.x; i < LC_HBINS; i += blockDim.x) hs[i] = 0;
    __syncthreads();
    const uint32_t hb = nbins < LC_HBINS ? nbins : LC_HBINS;
    uint32_t tot[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) tot[k] = 0;
    auto count = [&](uint32_t code, unsigned long long &A, unsigned long long &B) {
        const uint32_t idx = code - 1u;
        const unsigned long long one = 1ull << ((idx & 7u) * 8u);
        A += idx < 8u ? one : 0ull;
        B += idx - 8u < 8u ? one : 0ull;
        if (idx >= 16u) {
            if (code < hb) atomicAdd(&hs[code], 1u);
            else atomicAdd(&hist[code], 1u);
        }
    };
    auto flush = [&](unsigned long long A, unsigned long long B) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            tot[k] += (uint32_t)((A >> (8 * k)) & 0xffull);
            tot[8 + k] += (uint32_t)((B >> (8 * k)) & 0xffull);
        }
    };
    const uint64_t nv = m / 8;                                    // whole 16-byte vectors
    const uint4 *v4 = reinterpret_cast<const uint4 *>(codes);    // codes buffer is 16-byte aligned
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    while (i < nv) {
        unsigned long long A = 0ull, B = 0ull;
        for (int r = 0; r < 16 && i < nv; ++r, i += stride) {     // <= 128 codes per byte counter
            const uint4 q = __ldcs(v4 + i);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                count(w[h] & 0xffffu, A, B);
                count(w[h] >> 16, A, B);
            }
        }
        flush(A, B);
    }
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)(m - nv * 8)) {   // tail codes
        unsigned long long A = 0ull, B = 0ull;
        count(codes[nv * 8 + threadIdx.x], A, B);
        flush(A, B);
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 16; ++k) tot[k] = __reduce_add_sync(0xffffffffu, tot[k]);
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (lane == k) mine = tot[k];
    __syncthreads();
    if (lane < 16 && mine) {
        const uint32_t code = (uint32_t)lane + 1u;
        if (code < hb) atomicAdd(&hs[code], mine);
        else atomicAdd(&hist[code], mine);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < hb; k += blockDim.x)
        if (hs[k]) atomicAdd(&hist[k], hs[k]);
}

template __global__ void lc_quant_serial_kernel<uint16_t>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_serial_kernel<uint32_t>(LcQuantParams, uint32_t *);
template __global__ void lc_hist_kernel<uint16_t>(const uint16_t *, uint64_t, uint32_t *, uint32_t);
template __global__ void lc_hist_kernel<uint32_t>(const uint32_t *, uint64_t, uint32_t *, uint32_t);
