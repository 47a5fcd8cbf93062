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

// Lattice guess for the chain value at position pos given an anchor.
__device__ __forceinline__ double lc_guess(const LcQuantParams &P, double xpos, long long pos,
                                           long long apos, double aval)
{
    if (apos == pos) return aval;
    // a guess only has to be near the chain (the offset maps carry the rest), and chunk
    // c's end guess and chunk c+1's start guess come from identical inputs: RN(1/delta)
    // instead of a division
    const double k = floor(LC_ADD(LC_MUL(LC_SUB(xpos, aval), P.Q.inv), 0.5));
    if (k == 0.0) return aval;
    const double g = LC_ADD(aval, LC_MUL(k, P.Q.delta));
    return isfinite(g) ? g : xpos;
}

// ---------------------------------------------------------------------------
// Split quantizer: pass 0 (anchors, only when escapes are possible), pass A
// (guess chains + maps + in-tile scan), map scan over tiles, pass B (exact
// chain).  No tile ever waits for another tile.

// Load one tile of x into padded smem rows; xhalo[LC_L] = x[tile start].
// Coalesced 8-byte cp.async copies (no register staging: all 32 per thread are
// in flight at once); the caller publishes the tile with lc_cp_async_wait()
// + __syncthreads().  lc_prefetch_x_tile warms L2 with the tile a CTA
// processes next while it computes the current one.
__device__ __forceinline__ void lc_load_x_tile(const LcQuantParams &P, long long pbeg, double *xs, double *xhalo)
{
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    // element off = k * LC_TPB + tid goes to row off / 32, column off % 32: both
    // addresses advance by a constant per k (immediate offsets, no per-copy math)
    double *dst = xs + (tid >> 5) * LC_ROW + (tid & 31);
    const double *src = P.x + pbeg + 1 + tid;
    if (pbeg + LC_TILE <= nel) {                         // full tile
#pragma unroll
        for (int k = 0; k < LC_L; ++k) lc_cp_async8(dst + k * (LC_TPB / 32) * LC_ROW, src + k * LC_TPB);
    } else {
#pragma unroll
        for (int k = 0; k < LC_L; ++k)
            if (pbeg + 1 + k * LC_TPB + tid <= nel) lc_cp_async8(dst + k * (LC_TPB / 32) * LC_ROW, src + k * LC_TPB);
    }
    lc_cp_async_commit();
    if (tid <= LC_L) {
        const long long pos = pbeg - LC_L + tid;
        xhalo[tid] = pos >= 0 ? P.x[pos] : 0.0;
    }
}

__device__ __forceinline__ void lc_prefetch_x_tile(const LcQuantParams &P, long long t_next)
{
    if (t_next >= P.ntiles) return;
    const long long pbeg = (P.first_chunk + t_next * LC_TPB) * LC_L;
    const long long nel = (long long)P.n - 1;
    // LC_TILE doubles = 512 lines of 128 B: two per thread
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const long long pos = pbeg + 1 + (long long)(k * LC_TPB + threadIdx.x) * 16;
        if (pos <= nel) lc_prefetch_l2(P.x + pos);
    }
}

__global__ void __launch_bounds__(LC_TPB) lc_anchor_tiles_kernel(LcQuantParams P)
{
    if (!lc_quant_dyn(P) || !P.use_anchors) return;
    // last definite escape position of every tile (escapes certain from the data)
    __shared__ long long wmax[LC_TPB / 32];
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long pbeg = (P.first_chunk + t * LC_TPB) * LC_L;
        long long last = -1;
        for (int k = 0; k < LC_L; ++k) {
            const long long pos = pbeg + 1 + k * LC_TPB + tid;
            if (pos <= nel && lc_definite_escape(P.x[pos], P.x[pos - 1], P)) last = max(last, pos);
        }
        for (int o = 16; o; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        if ((tid & 31) == 0) wmax[tid >> 5] = last;
        __syncthreads();
        if (tid == 0) {
            for (int w = 0; w < LC_TPB / 32; ++w) last = max(last, wmax[w]);
            P.tile_last_esc[t] = last;
        }
        __syncthreads();
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

__global__ void __launch_bounds__(LC_TPB, 3) lc_quant_a_kernel(LcQuantParams P)
{
    if (!lc_quant_dyn(P)) return;
    typedef cub::BlockScan<long long, LC_TPB> ScanLL;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    double *xs = reinterpret_cast<double *>(lc_dyn_smem);
    __shared__ double xhalo[LC_L + 1];
    __shared__ typename ScanLL::TempStorage scan_tmp;
    __shared__ OffMap warp_agg[LC_TPB / 32];
    __shared__ LcReplayItem s_rq[LC_TPB];
    __shared__ int s_rcnt[LC_TPB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long nel = (long long)P.n - 1;
    const long long launch_apos = P.first_chunk * LC_L;

    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long pbeg = cbeg * LC_L;
        const long long c = cbeg + tid;
        const long long p0 = c * LC_L;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - p0) : 0;
        __syncthreads();
        lc_load_x_tile(P, pbeg, xs, xhalo);
        lc_cp_async_wait();
        __syncthreads();
        lc_prefetch_x_tile(P, t + gridDim.x);
        const double *row = xs + tid * LC_ROW;
        const double xstart = tid == 0 ? xhalo[LC_L] : xs[(tid - 1) * LC_ROW + LC_L - 1];

        // anchors
        long long apos, apos_next;
        if (P.use_anchors) {
            long long last_esc = -1;
            double xp = xstart;
            for (int j = 0; j < len; ++j) {
                const double xi = row[j];
                if (lc_definite_escape(xi, xp, P)) last_esc = p0 + 1 + j;
                xp = xi;
            }
            struct MaxOp { __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; } };
            long long esc_excl;
            ScanLL(scan_tmp).ExclusiveScan(last_esc, esc_excl, -1LL, MaxOp());
            const long long in = P.anc_in[t];
            apos = max(in, esc_excl);
            apos_next = max(apos, last_esc);
        } else {
            apos = apos_next = launch_apos;
        }
        // the launch anchor is x[0] itself on a fresh run (first_chunk 0)
        const bool relaunch = P.first_chunk != 0;
        const double aval = (relaunch && apos == launch_apos) ? P.anchor_val : P.x[apos];
        const double aval_next = (relaunch && apos_next == launch_apos) ? P.anchor_val : P.x[apos_next];
        const double xend = len > 0 ? row[len - 1] : xstart;
        const double g0 = lc_guess(P, xstart, p0, apos, aval);
        const double g1 = lc_guess(P, xend, p0 + len, apos_next, aval_next);

        // guess chain with superset event flags (lc_flags_*); flagged chunks are
        // replayed below by a compacted queue of threads
        OffMap H;
        bool need = false;
        unsigned mask = 0u;
        double r = g0, rs = g0;                      // rs: chain value before the first flagged step
        if (len > 0) {
            LcFlags F;
            lc_flags_init(F, g0);
            int anyesc = 0;
            for (int j = 0; j < len; ++j) {
                int esc; double inc;
                const double rn = lc_step_guess(P.Q, row[j], r, &esc, &inc);
                anyesc |= esc;
                const bool f = lc_flag_test(F, r, inc, rn);
                rs = (f && F.mask == 0u) ? r : rs;
                F.mask |= (unsigned)f << (j & 31);
                r = rn;
            }
            if (anyesc) H = lc_map_const(0.0);
            else {
                H = lc_map_identity(lc_ulp(g0));
                mask = F.mask;
                need = mask != 0u;
            }
        } else {
            H = lc_map_neutral();
        }
        lc_tile_replay(need, mask, g0, rs, s_rq, s_rcnt, [&](const LcReplayItem &it) {
            double *rw = xs + lc_replay_ch(it) * LC_ROW;
            const int j0 = __ffs(it.mask) - 1, j1 = 31 - __clz(it.mask);
            OffMap Hr = lc_map_identity(lc_replay_ulp(it));
            double r2 = it.rs;
            for (int j = j0; j <= j1; ++j) {
                int esc; double inc;
                const double rn = lc_step_guess(P.Q, rw[j], r2, &esc, &inc);
                if (((it.mask >> j) & 1u) && inc != 0.0) lc_map_step(Hr, r2, inc, rn);
                r2 = rn;
            }
            lc_map_to_words(reinterpret_cast<uint32_t *>(rw), Hr);
        });
        if (need) H = lc_map_from_words(reinterpret_cast<const uint32_t *>(row));
        if (len > 0 && c + 1 < P.nchunks) lc_map_shift_out(H, LC_SUB(r, g1));

        // in-tile inclusive scan of maps
        OffMap inc_map = H;
        lc_warp_scan_maps(inc_map);
        if (lane == 31) warp_agg[wid] = inc_map;
        __syncthreads();
        lc_scan_warp_maps(warp_agg, LC_TPB / 32);
        __syncthreads();
        if (wid > 0) inc_map = lc_map_compose(inc_map, warp_agg[wid - 1]);
        OffMap exc_map = lc_shfl_up_map(inc_map, 1);
        if (lane == 0) exc_map = wid > 0 ? warp_agg[wid - 1] : lc_map_neutral();
        if (len > 0) {
            P.pred.kind[c] = exc_map.kind;
            P.pred.B[c] = exc_map.B;
            P.pred.t0[c] = exc_map.t0;
            P.pred.t1[c] = exc_map.t1;
            P.pred.y[c] = exc_map.y;
            P.pred.g0[c] = g0;
        }
        if (tid == 0) P.tile_agg[t] = warp_agg[LC_TPB / 32 - 1];
    }
}

// Offsets at every tile start: D_0 = 0, D_{t+1} = agg_t(D_t).  G co-resident
// CTAs of 1024 threads (G <= SM count); thread i composes `per` consecutive tile
// maps, a block scan gives each thread's in-group exclusive map and the group
// aggregate, which is published (release flag).  Thread 0 folds the aggregates
// of all earlier groups (acquire; they never wait on later groups) into the
// offset at the group start; every thread then evaluates its tiles.
__global__ void __launch_bounds__(1024) lc_map_scan_kernel(const OffMap *__restrict__ agg, double *__restrict__ tileD,
                                                          long long ntiles, long long per, OffMap *gagg, int *gflag)
{
    __shared__ OffMap wsum[32];
    __shared__ double s_D;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, g = blockIdx.x;
    const long long b0 = min(ntiles, ((long long)g * 1024 + tid) * per), b1 = min(ntiles, b0 + per);
    OffMap run = lc_map_neutral();
    for (long long t = b0; t < b1; ++t) run = lc_map_compose(agg[t], run);
    OffMap inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const OffMap up = lc_shfl_up_map(inc, o);
        if (lane >= o) inc = lc_map_compose(inc, up);
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    lc_scan_warp_maps(wsum, 32);
    __syncthreads();
    if (wid > 0) inc = lc_map_compose(inc, wsum[wid - 1]);
    OffMap exc = lc_shfl_up_map(inc, 1);
    if (lane == 0) exc = wid > 0 ? wsum[wid - 1] : lc_map_neutral();
    if (tid == 0) {
        gagg[g] = wsum[31];
        __threadfence();
        st_release(gflag + g, 1);
        double D = 0.0;
        for (int j = 0; j < g; ++j) {
            while (ld_acquire(gflag + j) != 1) { }
            D = lc_map_eval(gagg[j], D);
        }
        s_D = D;
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
                       cudaStream_t st)
{
    long long G = (ntiles + 1023) / 1024;
    if (G > sm_count) G = sm_count;
    if (G > LC_MAPSCAN_MAXG) G = LC_MAPSCAN_MAXG;
    if (G < 1) G = 1;
    const long long per = (ntiles + 1024 * G - 1) / (1024 * G);
    OffMap *gagg = (OffMap *)scratch;
    int *gflag = (int *)(gagg + LC_MAPSCAN_MAXG);
    cudaError_t e = cudaMemsetAsync(gflag, 0, G * sizeof(int), st);
    if (e != cudaSuccess) return (int)e;
    lc_map_scan_kernel<<<(int)G, 1024, 0, st>>>(agg, tileD, ntiles, per, gagg, gflag);
    return (int)cudaGetLastError();
}

template <typename CodeT, bool REC>
__global__ void __launch_bounds__(LC_TPB, 3) lc_quant_b_kernel(LcQuantParams P, CodeT *__restrict__ codes)
{
    if (!lc_quant_dyn(P)) return;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    double *xs = reinterpret_cast<double *>(lc_dyn_smem);
    uint32_t *hs = reinterpret_cast<uint32_t *>(xs + LC_TPB * LC_ROW);
    __shared__ double xhalo[LC_L + 1];
    __shared__ double starts[LC_TPB + 1];
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    const uint32_t hb = P.nbins < LC_HBINS_B ? P.nbins : LC_HBINS_B;
    for (uint32_t i = tid; i < LC_HBINS_B; i += LC_TPB) hs[i] = 0;

    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long pbeg = cbeg * LC_L;
        const long long c = cbeg + tid;
        const long long p0 = c * LC_L;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - p0) : 0;
        __syncthreads();
        lc_load_x_tile(P, pbeg, xs, xhalo);
        const double Dt = P.tile_D[t];
        double start = 0.0;
        if (len > 0) {
            OffMap m;
            m.kind = P.pred.kind[c]; m.B = P.pred.B[c]; m.t0 = P.pred.t0[c]; m.t1 = P.pred.t1[c]; m.y = P.pred.y[c];
            m.v = 0.0; m.og = 0.0;
            start = lc_apply_offset(P.pred.g0[c], lc_map_eval(m, Dt));
            // test hook (LC_OPT_INJECT_QUANT): a wrong prediction, so the predecessor's end check fails
            if (c == P.inject_chunk && P.first_chunk == 0) start = lc_from_bits(lc_bits(start) ^ 1);
        }
        starts[tid] = start;
        if (tid == LC_TPB - 1) {
            const long long cn = cbeg + LC_TPB;          // first chunk of the next tile
            starts[LC_TPB] = (cn < P.nchunks) ? lc_apply_offset(P.pred.g0[cn], P.tile_D[t + 1]) : 0.0;
        }
        lc_cp_async_wait();
        __syncthreads();
        lc_prefetch_x_tile(P, t + gridDim.x);
        if (t + gridDim.x < P.ntiles) {                      // next tile's chunk predictions
            const long long cn = P.first_chunk + (t + gridDim.x) * LC_TPB;
            lc_prefetch_bytes(P.pred.kind + cn, LC_TPB * sizeof(int));
            lc_prefetch_bytes(P.pred.B + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(P.pred.t0 + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(P.pred.t1 + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(P.pred.y + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(P.pred.g0 + cn, LC_TPB * sizeof(double));
        }
        const double *row = xs + tid * LC_ROW;
        {
            double r = start;
            uint32_t *crow = reinterpret_cast<uint32_t *>(xs + tid * LC_ROW);
            bool ok = true;
            for (int j = 0; j < len; ++j) {
                uint32_t code; int esc; double inc, pe;
                const double rn = lc_step_nb(P.Q, row[j], r, &code, &inc, &esc, &pe, ok);
                crow[j] = code;
                if (REC) {
                    P.pe[p0 + j] = pe;
                    P.pe_rec[p0 + j] = LC_SUB(rn, r);
                }
                r = rn;
            }
            if (!ok) {                                        // a quotient was not certified: IEEE path
                r = start;
                for (int j = 0; j < len; ++j) {
                    uint32_t code; int esc; double inc, pe;
                    const double rn = lc_step(P.Q, P.x[p0 + 1 + j], r, &code, &esc, &inc, &pe);
                    crow[j] = code;
                    if (REC) {
                        P.pe[p0 + j] = pe;
                        P.pe_rec[p0 + j] = LC_SUB(rn, r);
                    }
                    r = rn;
                }
            }
            if (len > 0 && c + 1 < P.nchunks && lc_bits(r) != lc_bits(starts[tid + 1])) {
                P.bad_end[c] = r;
                atomicMin(P.first_bad, (unsigned long long)(c + 1));
            }
        }
        // histogram: codes 1..16 (the small |m| that dominate smooth data) in
        // packed per-thread byte counters (a chunk adds at most 32 to a code),
        // summed per warp with redux.sync; every other code atomically
        if (P.count_hist) {
            const uint32_t *crow = reinterpret_cast<const uint32_t *>(xs + tid * LC_ROW);
            unsigned long long A = 0ull, B = 0ull;
            for (int j = 0; j < len; ++j) {
                const uint32_t code = crow[j];
                const uint32_t idx = code - 1u;                   // escape (code 0) -> 2^32 - 1
                const unsigned long long one = 1ull << ((idx & 7u) * 8u);
                A += idx < 8u ? one : 0ull;
                B += idx - 8u < 8u ? one : 0ull;
                if (idx >= 16u) {
                    if (code < hb) atomicAdd(&hs[code], 1u);
                    else atomicAdd(&P.hist[code], 1u);
                }
            }
            uint32_t w[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                w[k] = (uint32_t)((A >> (16 * k)) & 0xffull) | ((uint32_t)((A >> (16 * k + 8)) & 0xffull) << 16);
                w[4 + k] = (uint32_t)((B >> (16 * k)) & 0xffull) | ((uint32_t)((B >> (16 * k + 8)) & 0xffull) << 16);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = __reduce_add_sync(0xffffffffu, w[k]);   // halves <= 1024
            // lane L < 16 adds the warp's count of code L + 1 (one atomic per lane, in parallel)
            const int lane = tid & 31;
            uint32_t mine = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if ((lane >> 1) == k) mine = (lane & 1) ? (w[k] >> 16) : (w[k] & 0xffffu);
            if (lane < 16 && mine) {
                const uint32_t code = (uint32_t)lane + 1u;
                if (code < hb) atomicAdd(&hs[code], mine);
                else atomicAdd(&P.hist[code], mine);
            }
        }
        __syncthreads();
        // coalesced 16-byte code stores: 16 / sizeof(CodeT) consecutive codes per thread
        {
            constexpr int V = 16 / sizeof(CodeT);
            const long long tile_n = min((long long)LC_TILE, nel - pbeg);
            for (int g = tid; g * V < tile_n; g += LC_TPB) {
                const int off = g * V;                       // first element of the group
                const uint32_t *src = reinterpret_cast<const uint32_t *>(xs) + (off >> 5) * (2 * LC_ROW) + (off & 31);
                if (off + V <= tile_n) {
                    uint4 v;
                    if (V == 8) {
                        v.x = (src[0] & 0xffffu) | (src[1] << 16);
                        v.y = (src[2] & 0xffffu) | (src[3] << 16);
                        v.z = (src[4] & 0xffffu) | (src[5] << 16);
                        v.w = (src[6] & 0xffffu) | (src[7] << 16);
                    } else {
                        v.x = src[0]; v.y = src[1]; v.z = src[2]; v.w = src[3];
                    }
                    *reinterpret_cast<uint4 *>(codes + pbeg + off) = v;
                } else {
                    for (int k = 0; off + k < tile_n; ++k) codes[pbeg + off + k] = (CodeT)src[k];
                }
            }
        }
    }
    __syncthreads();
    if (P.count_hist)
        for (uint32_t i = tid; i < hb; i += LC_TPB)
            if (hs[i]) atomicAdd(&P.hist[i], hs[i]);
}

size_t lc_quant_a_smem_bytes() { return sizeof(double) * LC_TPB * LC_ROW; }
size_t lc_quant_b_smem_bytes() { return sizeof(double) * LC_TPB * LC_ROW + sizeof(uint32_t) * LC_HBINS_B; }

template __global__ void lc_quant_b_kernel<uint16_t, false>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_b_kernel<uint32_t, false>(LcQuantParams, uint32_t *);
template __global__ void lc_quant_b_kernel<uint16_t, true>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_b_kernel<uint32_t, true>(LcQuantParams, uint32_t *);

// Sequential exact chain from chunk `first_chunk` (fallback for inputs whose
// chunk predictions keep failing).  One thread; correct for every input.
template <typename CodeT>
__global__ void lc_quant_serial_kernel(LcQuantParams P, CodeT *__restrict__ codes)
{
    if (!lc_quant_dyn(P)) return;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double r = P.anchor_val;
    for (uint64_t i = (uint64_t)P.first_chunk * LC_L + 1; i < P.n; ++i) {
        uint32_t code; int esc; double inc, pe;
        const double rn = lc_step(P.Q, P.x[i], r, &code, &esc, &inc, &pe);
        codes[i - 1] = (CodeT)code;
        if (P.pe) { P.pe[i - 1] = pe; P.pe_rec[i - 1] = LC_SUB(rn, r); }
        r = rn;
    }
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
