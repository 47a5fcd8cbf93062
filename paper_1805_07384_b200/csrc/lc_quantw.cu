// lc_quantw.cu -- exact quantizer in one streaming pass over x (sm_100a).
//
// Replaces the sequential _compress_kernel (compressor.py:319-355) and
// np.bincount (compressor.py:411).  In the common case every x element is read
// from HBM once and every code written once; the histogram is counted where
// the codes are produced.
//
// Work unit: a WARP TILE of 32 chunks x 32 elements (one chunk per lane).  Warps
// never wait for each other (no CTA barriers), so the dependent FP64 chains of
// different warps hide each other's latency.
//
//   lc_quant_wa_kernel (pass A, per warp tile):
//     * x tile -> the warp's shared-memory rows (coalesced cp.async);
//     * guess chain per chunk from the lattice guess g0 (lc_chain.cuh): the
//       reference step with pe * RN(1/delta) in place of pe / delta.  Each step
//       emits its code (staged in shared memory, stored coalesced), counts it in
//       the histogram, flags possible offset-map events and tracks the chunk's
//       decision margin amax = max |frac(qq) - 1/2|;
//     * flagged lanes replay their chunk to build its offset map; a warp scan
//       composes the maps; the warp-tile aggregate goes to tile_agg[w];
//     * certification slack S_w: the guess codes of chunk c are the reference's
//       whenever |D_w| < S_c, where D_w is the exact offset (true - guess) at the
//       warp-tile start, so S_w = min_c S_c (see lc_qw_slack).
//   lc_map_scan_kernel: exact offsets D_w at every warp-tile start.
//   lc_quant_wfix_kernel (per warp tile): |D_w| < S_w -> nothing to do (the
//     common case: two loads).  Otherwise the warp redoes pass A for its tile,
//     certifies chunk by chunk with the exact D_c, re-runs the uncertified
//     chunks with the exact reference step from their predicted start (codes
//     and histogram entries replaced) and checks each re-run chunk's exact end
//     against the next chunk's predicted start.  The first failure triggers a
//     host relaunch from that chunk with its exact start.  By induction from
//     the launch anchor every chunk before the first failure had an exact
//     predicted start (no decision differed before it), so its codes --
//     certified or re-run -- are the reference's.
//
// Certification.  True chain = guess chain + D; D starts
// at D_c and moves by at most ulp(Rmax) <= 2^-52 Rmax per step (both chains'
// values are bounded by Rmax = (max|x| + eb)(1 + 2^-50)).  If
//     |D_c| + len * 2^-52 Rmax < M_c = (1/2 - amax - 5T) delta (1 - 2^-40) - 2^-48 (Rmax + eb)
// (T: the tolerance of lc_step_nb's certified decision; amax = max over the
// chunk's steps of |RN(pe * RN(1/delta)) - floor(qq)|, within T/4 of
// |frac(qq) - 1/2|), every step takes the
// reference's decision m and its |x - cand| <= eb test agrees: the codes are
// the reference's.
#include "lc_kernels.cuh"

#define LC_QW_ROWS (32 * LC_ROW)       // doubles of one warp's x tile (padded rows)
#define LC_QW_CW 34                     // u16 code staging row (17 words: odd stride)

__device__ __forceinline__ bool lc_qw_dyn(LcQuantParams &P)
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
    P.rmax = __ldg(&d->rmax);
    return true;
}

__device__ __forceinline__ bool lc_qw_definite_escape(double xi, double xprev, const LcQuantParams &P)
{
    const double d = fabs(LC_SUB(xi, xprev));
    return LC_SUB(LC_MUL(d, 1.0 - 0x1p-50), LC_MUL(P.Q.eb, 1.0 + 0x1p-50)) >= P.esc_thresh;
}

// Lattice guess for the chain value at position pos given an anchor: only has
// to be near the chain (the offset maps carry the rest); chunk c's end guess and
// chunk c+1's start guess come from identical inputs.
__device__ __forceinline__ double lc_qw_guess(const LcQuantParams &P, double xpos, long long pos, long long apos,
                                              double aval)
{
    if (apos == pos) return aval;
    const double k = floor(LC_ADD(LC_MUL(LC_SUB(xpos, aval), P.Q.inv), 0.5));
    if (k == 0.0) return aval;
    const double g = LC_ADD(aval, LC_MUL(k, P.Q.delta));
    return isfinite(g) ? g : xpos;
}

// Histogram increments of codes 1..16 as byte counters (code k+1 -> byte k % 4 of
// word k / 4); entry 16 (escapes and codes > 16) is zero.
__constant__ uint4 c_qw_hinc[17] = {
    {1u, 0, 0, 0}, {1u << 8, 0, 0, 0}, {1u << 16, 0, 0, 0}, {1u << 24, 0, 0, 0},
    {0, 1u, 0, 0}, {0, 1u << 8, 0, 0}, {0, 1u << 16, 0, 0}, {0, 1u << 24, 0, 0},
    {0, 0, 1u, 0}, {0, 0, 1u << 8, 0}, {0, 0, 1u << 16, 0}, {0, 0, 1u << 24, 0},
    {0, 0, 0, 1u}, {0, 0, 0, 1u << 8}, {0, 0, 0, 1u << 16}, {0, 0, 0, 1u << 24},
    {0, 0, 0, 0}};

__device__ __forceinline__ void lc_qw_hist_add(uint32_t *hs, uint32_t *hist, uint32_t hb, uint32_t code, uint32_t v)
{
    if (code < hb) atomicAdd(&hs[code], v);
    else atomicAdd(&hist[code], v);
}

// Per-lane state of pass A on one warp tile.
struct LcQwLane {
    long long c, p0;    // chunk index, position of the chunk start value
    int len;            // codes of the chunk (0: past the end)
    double g0, g1;      // guesses at the chunk start / end
    double amax;        // max |RN(pe * inv) - floor(qq)| over the chunk's steps
    OffMap H;           // chunk map (offset at start -> offset at the next chunk's guess)
    OffMap inc, exc;    // inclusive / exclusive warp scans of the maps
};

// Pass A on warp tile w (all 32 lanes).  xw: the warp's x rows; cw (optional):
// the warp's code staging rows, hs/hist (optional): histogram.
template <typename CodeT, bool EMIT>
__device__ __forceinline__ void lc_qw_pass_a(const LcQuantParams &P, long long w, double *xw, uint16_t *cw,
                                             uint32_t *hs, uint32_t hb, const uint4 *hinc, LcQwLane &L)
{
    const int lane = threadIdx.x & 31;
    const long long nel = (long long)P.n - 1;
    const long long wc0 = P.first_chunk + w * 32;            // first chunk of the warp tile
    const long long pbeg = wc0 * LC_L;
    L.c = wc0 + lane;
    L.p0 = L.c * LC_L;
    L.len = (L.c < P.nchunks) ? (int)min((long long)LC_L, nel - L.p0) : 0;
    const int len = L.len;
    // x tile: element e = k * 32 + lane -> row k (chunk), column lane
    {
        const double *src = P.x + pbeg + 1 + lane;
        double *dst = xw + lane;
        if (pbeg + 32 * LC_L <= nel) {
#pragma unroll
            for (int k = 0; k < 32; ++k) lc_cp_async8(dst + k * LC_ROW, src + k * 32);
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (pbeg + 1 + k * 32 + lane <= nel) lc_cp_async8(dst + k * LC_ROW, src + k * 32);
        }
        lc_cp_async_commit();
    }
    const double xprev_tile = P.x[pbeg];                      // value at the tile's first chunk start
    lc_cp_async_wait();
    __syncwarp();
    const double *row = xw + lane * LC_ROW;
    const double xlast_prev = __shfl_up_sync(0xffffffffu, len > 0 ? row[LC_L - 1] : 0.0, 1);
    const double xstart = lane == 0 ? xprev_tile : xlast_prev;
    const long long launch_apos = P.first_chunk * LC_L;
    long long apos, apos_next;
    if (P.use_anchors) {
        long long last_esc = -1;
        double xp = xstart;
        for (int j = 0; j < len; ++j) {
            const double xi = row[j];
            if (lc_qw_definite_escape(xi, xp, P)) last_esc = L.p0 + 1 + j;
            xp = xi;
        }
        long long incl = last_esc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long up = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = max(incl, up);
        }
        long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = -1;
        apos = max(P.anc_in[w], excl);
        apos_next = max(apos, last_esc);
    } else {
        apos = apos_next = launch_apos;
    }
    const bool relaunch = P.first_chunk != 0;
    const double aval = (relaunch && apos == launch_apos) ? P.anchor_val : P.x[apos];
    const double aval_next = (relaunch && apos_next == launch_apos) ? P.anchor_val : P.x[apos_next];
    const double xend = len > 0 ? row[len - 1] : xstart;
    L.g0 = lc_qw_guess(P, xstart, L.p0, apos, aval);
    L.g1 = lc_qw_guess(P, xend, L.p0 + len, apos_next, aval_next);

    // guess chain: codes, histogram, event flags, decision margin
    bool need = false;
    double r = L.g0;
    double amax = 0.0;                                   // max |RN(pe * inv) - fq| (~ |frac(qq) - 1/2|)
    uint32_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;             // byte counters of codes 1..16 (4 per word)
    bool anybig = false;
    uint32_t maxc = 0;                                   // largest code of the chunk
    uint16_t *crow = nullptr;
    uint32_t *crow32 = nullptr;
    if (len > 0) {
        LcFlags F;
        lc_flags_init(F, L.g0);
        bool anyesc = false, anyf = false;
        crow = cw + lane * LC_QW_CW;
        crow32 = reinterpret_cast<uint32_t *>(cw) + lane * 33;
        auto body = [&](int j) {
            const double v = row[j];
            const double pe = LC_SUB(v, r);
            const double u = LC_MUL(pe, P.Q.inv);
            const double fq = floor(LC_ADD(u, 0.5));
            const double inc = LC_MUL(fq, P.Q.delta);
            const double cand = LC_ADD(r, inc);
            const bool keep = fabs(fq) <= P.Q.max_m && fabs(LC_SUB(v, cand)) <= P.Q.eb;
            const double rn = keep ? cand : v;
            const double a = fabs(LC_SUB(u, fq));
            amax = a > amax ? a : amax;
            if (EMIT) {
                const int m = (int)(uint32_t)(lc_bits(LC_ADD(fq, 6755399441055744.0)) & 0xffffffffLL);
                const uint32_t code = keep ? (((uint32_t)m << 1) ^ (uint32_t)(m >> 31)) + 1u : 0u;
                if (sizeof(CodeT) == 2) crow[j] = (uint16_t)code;
                else crow32[j] = code;
                const uint32_t idx = min(code - 1u, 16u);    // escape (0) and codes > 16 -> zero entry
                const uint4 e = hinc[idx];           // shared memory: same code -> broadcast
                h0 += e.x; h1 += e.y; h2 += e.z; h3 += e.w;
                anybig |= code - 1u >= 16u;          // escapes and codes > 16: counted after the chain
                maxc = code > maxc ? code : maxc;
            }
            anyesc |= !keep;
            anyf |= lc_flag_test(F, r, inc, rn);
            r = rn;
        };
#pragma unroll 4
        for (int j = 0; j < len; ++j) body(j);
        if (anyesc) L.H = lc_map_const(0.0);
        else {
            L.H = lc_map_identity(lc_ulp(L.g0));
            need = anyf;
        }
    } else {
        L.H = lc_map_neutral();
    }
    L.amax = amax;
    if (EMIT) {   // warp totals of codes 1..16 (a chunk adds at most 32 per code)
        const uint32_t hw[4] = {h0, h1, h2, h3};
        uint32_t wsum[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            wsum[2 * k] = __reduce_add_sync(0xffffffffu, hw[k] & 0x00ff00ffu);          // codes 4k+1, 4k+3
            wsum[2 * k + 1] = __reduce_add_sync(0xffffffffu, (hw[k] >> 8) & 0x00ff00ffu); // codes 4k+2, 4k+4
        }
        // lane L < 16 owns code L + 1: word L / 4, byte L % 4
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (lane == 4 * k + b) mine = (wsum[2 * k + (b & 1)] >> (16 * (b >> 1))) & 0xffffu;
        if (lane < 16 && mine) lc_qw_hist_add(hs, P.hist, hb, (uint32_t)lane + 1u, mine);
        {
            const uint32_t wm = __reduce_max_sync(0xffffffffu, maxc);
            if (lane == 0 && wm > hs[LC_HBINS_B + 1]) atomicMax(&hs[LC_HBINS_B + 1], wm);
        }
        // the other codes (escapes, |m| > 8): a second walk over the lane's staged row, outside
        // the dependent chain, so the (divergent) atomics pipeline instead of stalling it
        if (__any_sync(0xffffffffu, anybig)) {
            if (anybig) {
                unsigned nbig = 0;                   // codes beyond the shared-memory bins: lc_histw_kernel's
                if (sizeof(CodeT) == 2) {
                    const uint32_t *c2 = reinterpret_cast<const uint32_t *>(crow);   // rows start word aligned
#pragma unroll 4
                    for (int j = 0; j < len; j += 2) {
                        const uint32_t pr = c2[j >> 1];
                        const uint32_t ca = pr & 0xffffu, cb = pr >> 16;
                        if (ca - 1u >= 16u) { if (ca < hb) atomicAdd(&hs[ca], 1u); else ++nbig; }
                        if (j + 1 < len && cb - 1u >= 16u) { if (cb < hb) atomicAdd(&hs[cb], 1u); else ++nbig; }
                    }
                } else {
#pragma unroll 4
                    for (int j = 0; j < len; ++j) {
                        const uint32_t ca = crow32[j];
                        if (ca - 1u >= 16u) { if (ca < hb) atomicAdd(&hs[ca], 1u); else ++nbig; }
                    }
                }
                if (nbig) atomicAdd(&hs[LC_HBINS_B], nbig);   // the CTA's count, flushed with the histogram
            }
        }
    }
    // flagged lanes replay their chunk from its start, applying the exact step map
    // at every flagged step (a flagged non-event is a no-op)
    if (need) {
        LcFlags F;
        lc_flags_init(F, L.g0);
        OffMap Hr = lc_map_identity(lc_ulp(L.g0));
        double r2 = L.g0;
        for (int j = 0; j < len; ++j) {
            int esc; double inc;
            const double rn = lc_step_guess(P.Q, row[j], r2, &esc, &inc);
            if (inc != 0.0 && lc_flag_test(F, r2, inc, rn)) lc_map_step(Hr, r2, inc, rn);
            r2 = rn;
        }
        L.H = Hr;
    }
    if (len > 0 && L.c + 1 < P.nchunks) lc_map_shift_out(L.H, LC_SUB(r, L.g1));
    L.inc = L.H;
    lc_warp_scan_maps(L.inc);
    L.exc = lc_shfl_up_map(L.inc, 1);
    if (lane == 0) L.exc = lc_map_neutral();
}

// Upper bound of |H(D) - D| over all D (H periodic: y + kP + jump, |.| <= |y - t0| + 3B).
__device__ __forceinline__ double lc_qw_drift(const OffMap &H)
{
    if (H.kind == LC_MAP_TRANS) return fabs(H.y);
    if (H.kind == LC_MAP_PERIODIC) return LC_ADD(fabs(LC_SUB(H.y, H.t0)), LC_MUL(3.0, H.B));
    return INFINITY;
}

// The chunk's certification margin M_c minus the in-chunk drift bound.
__device__ __forceinline__ double lc_qw_margin(const LcQuantParams &P, const LcQwLane &L)
{
    const double T = LC_SUB(0.5, P.Q.cert);
    const double M = LC_SUB(LC_MUL(LC_SUB(LC_SUB(0.5, L.amax), LC_MUL(5.0, T)), LC_MUL(P.Q.delta, 1.0 - 0x1p-40)),
                            LC_MUL(LC_ADD(P.rmax, P.Q.eb), 0x1p-48));
    return LC_SUB(M, LC_MUL((double)L.len, LC_MUL(P.rmax, 0x1p-52)));
}

// Slack S_c: chunk c is certified for every tile offset D with |D| < S_c
// (|exc_c(D)| <= |D| + drift(exc_c); a constant exc map does not depend on D).
__device__ __forceinline__ double lc_qw_slack(const LcQuantParams &P, const LcQwLane &L)
{
    if (L.len == 0) return INFINITY;
    const double m = lc_qw_margin(P, L);
    if (L.exc.kind == LC_MAP_CONST) return fabs(L.exc.y) < m ? INFINITY : -INFINITY;
    const double s = LC_SUB(m, lc_qw_drift(L.exc));
    return s == s ? s : -INFINITY;                       // NaN -> never
}

template <typename CodeT>
__global__ void __launch_bounds__(LC_QW_TPB, 5) lc_quant_wa_kernel(LcQuantParams P, CodeT *__restrict__ codes)
{
    if (!lc_qw_dyn(P)) return;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int CWW = sizeof(CodeT) == 2 ? 32 * LC_QW_CW / 2 : 32 * 33;   // 32-bit words per warp
    double *xw = reinterpret_cast<double *>(lc_dyn_smem) + wid * LC_QW_ROWS;
    uint32_t *cw32 = reinterpret_cast<uint32_t *>(reinterpret_cast<double *>(lc_dyn_smem) + (LC_QW_TPB / 32) * LC_QW_ROWS)
                     + wid * CWW;
    uint32_t *hs = reinterpret_cast<uint32_t *>(reinterpret_cast<double *>(lc_dyn_smem) + (LC_QW_TPB / 32) * LC_QW_ROWS)
                   + (LC_QW_TPB / 32) * CWW;
    const long long nel = (long long)P.n - 1;
    const uint32_t hb = P.nbins < LC_HBINS_B ? P.nbins : LC_HBINS_B;
    for (uint32_t i = tid; i <= LC_HBINS_B + 1; i += LC_QW_TPB) hs[i] = 0;  // [LC_HBINS_B]: codes beyond the bins, [+1]: max code
    __shared__ uint4 s_hinc[17];
    if (tid < 17) s_hinc[tid] = c_qw_hinc[tid];
    __syncthreads();
    // vectors whose whole range lies below 2^-960 have subnormal ulps: the offset-map arithmetic
    // is not exact there, so nothing is certified (every chunk is re-run exactly and end-checked)
    // small bin budgets (n_bins_half < 1024): the chain cannot follow x, so it can sit far from the
    // guess lattice and the offsets stop being exactly representable (g + D off by an ulp: found by a
    // randomized run as wrong v3 sync starts at n_bins_half = 1 and 7): nothing is certified either
    const bool force = P.verify || P.pe != nullptr || !(P.rmax < INFINITY) || P.rmax < 0x1p-960 || P.nbins < 2048u ||
                       P.inject_chunk >= 0;
    // warp tiles are claimed by ticket (balanced tail); the next ticket is taken
    // one tile ahead so its x can be prefetched into L2 while this one runs
    long long w = 0, wnext = 0;
    if (lane == 0) w = (long long)atomicAdd(P.tile_counter, 1u);
    w = __shfl_sync(0xffffffffu, w, 0);
    for (; w < P.ntiles; w = wnext) {
        if (lane == 0) wnext = (long long)atomicAdd(P.tile_counter, 1u);
        wnext = __shfl_sync(0xffffffffu, wnext, 0);
        if (wnext < P.ntiles) {                            // 8 KB of x: two 128-byte lines per lane
            const long long pn = (P.first_chunk + wnext * 32) * LC_L + 1;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const long long pos = pn + (long long)(k * 32 + lane) * 16;
                if (pos <= nel) lc_prefetch_l2(P.x + pos);
            }
        }
        LcQwLane L;
        lc_qw_pass_a<CodeT, true>(P, w, xw, reinterpret_cast<uint16_t *>(cw32), hs, hb, s_hinc, L);
        // slack of the warp tile
        double s = force ? -INFINITY : lc_qw_slack(P, L);
#pragma unroll
        for (int o = 16; o; o >>= 1) s = fmin(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (lane == 31) P.tile_agg[w] = L.inc;
        if (lane == 0) { P.tile_S[w] = s; P.tile_g0[w] = L.g0; }
        // codes: coalesced 16-byte stores from the staging rows
        __syncwarp();
        const long long pbeg = (P.first_chunk + w * 32) * LC_L;
        const long long tile_n = min((long long)(32 * LC_L), nel - pbeg);
        constexpr int V = 16 / sizeof(CodeT);
        for (int g = lane; g * V < tile_n; g += 32) {
            const int off = g * V;
            if (sizeof(CodeT) == 2) {
                const uint32_t *s32 = cw32 + (off >> 5) * (LC_QW_CW / 2) + ((off & 31) >> 1);
                if (off + V <= tile_n) {
                    *reinterpret_cast<uint4 *>(codes + pbeg + off) = make_uint4(s32[0], s32[1], s32[2], s32[3]);
                } else {
                    const uint16_t *s16 = reinterpret_cast<const uint16_t *>(cw32) + (off >> 5) * LC_QW_CW + (off & 31);
                    for (int k = 0; off + k < tile_n; ++k) codes[pbeg + off + k] = (CodeT)s16[k];
                }
            } else {
                const uint32_t *s32 = cw32 + (off >> 5) * 33 + (off & 31);
                if (off + V <= tile_n) {
                    *reinterpret_cast<uint4 *>(codes + pbeg + off) = make_uint4(s32[0], s32[1], s32[2], s32[3]);
                } else {
                    for (int k = 0; off + k < tile_n; ++k) codes[pbeg + off + k] = (CodeT)s32[k];
                }
            }
        }
        __syncwarp();
    }
    __syncthreads();
    for (uint32_t i = tid; i < hb; i += LC_QW_TPB)
        if (hs[i]) atomicAdd(&P.hist[i], hs[i]);
    if (tid == 0 && hs[LC_HBINS_B]) atomicAdd(P.nbig, (unsigned long long)hs[LC_HBINS_B]);
    if (tid == 0 && hs[LC_HBINS_B + 1]) atomicMax(P.maxcode, hs[LC_HBINS_B + 1]);
}

// Exact reference chain of one chunk from `start` (certified decisions, IEEE
// division on doubt), codes and histogram entries replaced where they differ
// from what the chunk holds, end checked against `next` (the successor's
// predicted start): a mismatch records the first failing chunk.
template <typename CodeT, bool REC>
__device__ __forceinline__ void lc_qw_exact_chunk(const LcQuantParams &P, CodeT *__restrict__ codes,
                                                  const double *row, const LcQwLane &L, double start, double next)
{
    const long long q0 = L.p0;
    const int ln = L.len;
    double r2 = start;
    bool ok = true;
    for (int j = 0; j < ln; ++j) {
        uint32_t code; int esc; double inc, pe;
        const double rn = lc_step_nb(P.Q, row[j], r2, &code, &inc, &esc, &pe, ok);
        r2 = rn;
    }
    const bool ieee = !ok;
    r2 = start;
    for (int j = 0; j < ln; ++j) {                      // second run: write (same results when ok)
        uint32_t code; int esc; double inc, pe;
        bool ok2 = true;
        const double rn = ieee ? lc_step(P.Q, row[j], r2, &code, &esc, &inc, &pe)
                               : lc_step_nb(P.Q, row[j], r2, &code, &inc, &esc, &pe, ok2);
        const uint32_t old = (uint32_t)codes[q0 + j];
        if (old != code) {                              // bins >= LC_HBINS_B belong to lc_histw_kernel (final codes)
            const uint32_t hb = P.nbins < LC_HBINS_B ? P.nbins : LC_HBINS_B;
            if (old < hb) atomicAdd(&P.hist[old], 0xffffffffu);
            if (code < hb) atomicAdd(&P.hist[code], 1u);
            else atomicAdd(P.nbig, 1ull);
            atomicMax(P.maxcode, code);
            codes[q0 + j] = (CodeT)code;
        }
        if (REC) { P.pe[q0 + j] = pe; P.pe_rec[q0 + j] = LC_SUB(rn, r2); }
        r2 = rn;
    }
    if (L.c + 1 < P.nchunks && lc_bits(r2) != lc_bits(next)) {
        P.bad_end[L.c] = r2;
        atomicMin(P.first_bad, (unsigned long long)(L.c + 1));
    }
}

// Pass B.  P.resume = 0: the first pass over all warp tiles; a tile whose chunk
// codes get rewritten (modes 0 and 2) is marked (tile_S = -inf).  P.resume = 1 (one warp):
// resume at chunk P.resume_chunk, whose predicted start was wrong -- its exact
// start is known, so the chunks from there to the end of its warp tile are
// re-run exactly from offsets composed from that start (suffix scan of the
// tile's chunk maps, pass A recomputed), and the offset at the next tile start
// goes to *P.resume_D0 for the map scan of the remaining tiles.  P.resume = 2:
// the tiles after it with the new offsets; a tile marked in the first pass is
// re-run exactly in full (its codes came from wrong starts).  Pass A's codes,
// histogram, maps and slacks stay valid throughout (they do not depend on the
// offsets), so a failed prediction costs a map scan and this pass instead of a
// relaunch of the whole quantizer.
template <typename CodeT, bool REC>
__global__ void __launch_bounds__(LC_QW_TPB, 5) lc_quant_wfix_kernel(LcQuantParams P, CodeT *__restrict__ codes)
{
    if (!lc_qw_dyn(P)) return;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *xw = reinterpret_cast<double *>(lc_dyn_smem) + wid * LC_QW_ROWS;
    unsigned long long exact_chunks = 0;
    const bool force = P.verify || REC || !(P.rmax < INFINITY) || P.rmax < 0x1p-960 || P.nbins < 2048u || P.inject_chunk >= 0;
    if (P.resume == 1) {
        if (wid != 0) return;
        const long long rel = P.resume_chunk - P.first_chunk;
        const long long w = rel / 32;
        const int f0 = (int)(rel % 32);
        LcQwLane L;
        lc_qw_pass_a<CodeT, false>(P, w, xw, nullptr, nullptr, 0u, nullptr, L);
        OffMap sinc = lane >= f0 ? L.H : lc_map_neutral();
        lc_warp_scan_maps(sinc);
        OffMap sexc = lc_shfl_up_map(sinc, 1);
        if (lane <= f0) sexc = lc_map_neutral();
        const double exact = *P.resume_start;
        const double D0l = LC_SUB(exact, L.g0);
        const bool okl = lane == f0 && lc_bits(lc_apply_offset(L.g0, D0l)) == lc_bits(exact);
        const double D = __shfl_sync(0xffffffffu, D0l, f0);
        const bool ok = __shfl_sync(0xffffffffu, okl ? 1 : 0, f0) != 0;
        const double Dnext = lc_map_eval(sinc, D);       // lane 31: offset at the next tile start
        if (!ok) {                                       // offset not representable: full relaunch
            if (lane == 0) { *P.resume_D0 = NAN; atomicMin(P.first_bad, (unsigned long long)P.resume_chunk); }
            return;
        }
        double start = 0.0;
        if (lane >= f0 && L.len > 0) start = lane == f0 ? exact : lc_apply_offset(L.g0, lc_map_eval(sexc, D));
        double next = __shfl_down_sync(0xffffffffu, start, 1);
        if (lane == 31) next = lc_apply_offset(L.g1, Dnext);
        if (lane >= f0 && L.len > 0) {
            lc_qw_exact_chunk<CodeT, REC>(P, codes, xw + lane * LC_ROW, L, start, next);
            ++exact_chunks;
        }
        if (lane == 31) *P.resume_D0 = Dnext;
        if (f0 == 0 && lane == 0) P.tile_D[w] = D;       // the tile starts at the resumed chunk (v3 sync start)
        if (exact_chunks) atomicAdd(P.exact_count, exact_chunks);
        return;
    }
    if (P.resume == 2 && !(*P.resume_D0 == *P.resume_D0)) return;   // resume impossible (NaN)
    const long long nwarps = (long long)gridDim.x * (LC_QW_TPB / 32);
    // 32 warp tiles are checked per round (one per lane, coalesced loads); the
    // uncertified ones (rare) are then redone one after the other by the warp
    for (long long w0 = P.first_tile + ((long long)blockIdx.x * (LC_QW_TPB / 32) + wid) * 32; w0 < P.ntiles;
         w0 += nwarps * 32) {
        const long long wl = w0 + lane;
        const bool redo = wl < P.ntiles && !(fabs(P.tile_D[wl]) < P.tile_S[wl]);
        unsigned todo = __ballot_sync(0xffffffffu, redo);
      while (todo) {
        const long long w = w0 + __ffs(todo) - 1;
        todo &= todo - 1;
        const double Dw = P.tile_D[w];
        const bool marked = P.resume == 2 && P.tile_S[w] == -INFINITY;   // rewritten by the first pass
        LcQwLane L;
        lc_qw_pass_a<CodeT, false>(P, w, xw, nullptr, nullptr, 0u, nullptr, L);
        const double Dc = lc_map_eval(L.exc, Dw);
        double start = 0.0;
        if (L.len > 0) {
            start = lc_apply_offset(L.g0, Dc);
            // test hook (LC_OPT_INJECT_QUANT): a wrong prediction for this chunk
            if (L.c == P.inject_chunk && P.first_chunk == 0) start = lc_from_bits(lc_bits(start) ^ 1);
        }
        double next = __shfl_down_sync(0xffffffffu, start, 1);
        if (lane == 31) next = lc_apply_offset(L.g1, lc_map_eval(L.inc, Dw));
        const bool cert = !force && !marked && L.len > 0 && fabs(Dc) < lc_qw_margin(P, L);
        const bool rerun = L.len > 0 && !cert;
        if (rerun) {
            lc_qw_exact_chunk<CodeT, REC>(P, codes, xw + lane * LC_ROW, L, start, next);
            ++exact_chunks;
        }
        if (__any_sync(0xffffffffu, rerun) && lane == 0) P.tile_S[w] = -INFINITY;   // codes rewritten
        __syncwarp();
      }
    }
    if (exact_chunks) atomicAdd(P.exact_count, exact_chunks);
}

size_t lc_quantw_smem_bytes(int code_bytes)
{
    const size_t cww = code_bytes == 2 ? 32 * LC_QW_CW / 2 : 32 * 33;
    return sizeof(double) * LC_QW_TPB / 32 * LC_QW_ROWS + sizeof(uint32_t) * (LC_QW_TPB / 32) * cww +
           sizeof(uint32_t) * (LC_HBINS_B + 4);
}
size_t lc_quantw_fix_smem_bytes() { return sizeof(double) * LC_QW_TPB / 32 * LC_QW_ROWS; }

template __global__ void lc_quant_wa_kernel<uint16_t>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_wa_kernel<uint32_t>(LcQuantParams, uint32_t *);
template __global__ void lc_quant_wfix_kernel<uint16_t, false>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_wfix_kernel<uint32_t, false>(LcQuantParams, uint32_t *);
template __global__ void lc_quant_wfix_kernel<uint16_t, true>(LcQuantParams, uint16_t *);
template __global__ void lc_quant_wfix_kernel<uint32_t, true>(LcQuantParams, uint32_t *);
