// lc_common.cuh -- shared device helpers for the sm_100a codec kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "lc_chain.cuh"

#define LC_TPB 256                 // threads per block in the chunked kernels
#define LC_L 32                    // elements per chunk (one thread)
#define LC_TILE (LC_TPB * LC_L)    // codes per tile (8192)
#define LC_ROW (LC_L + 1)          // padded smem row (conflict-free column walk)
#define LC_HBINS 4096              // histogram bins privatised in smem
#define LC_HBINS_B 512             // ... in pass A (44.6 KB per CTA: five 4-warp CTAs per SM); larger codes: lc_histw_kernel

// Look-back descriptor of one tile (decoupled look-back, two channels:
// anchor positions and offset maps).
struct __align__(16) LcTileDesc {
    int st_anchor;                 // 0 none, 1 aggregate, 2 inclusive
    int st_map;
    long long anc_agg, anc_incl;   // last definite-escape position (max scan)
    int map_kind;
    int pad;
    double mv, mB, mt0, mt1, my, mog;  // aggregate OffMap
    double incl_D;                 // offset at the start of the next tile
};

__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void lc_store_map(LcTileDesc *d, const OffMap &m)
{
    d->map_kind = m.kind; d->mv = m.v; d->mB = m.B; d->mt0 = m.t0; d->mt1 = m.t1;
    d->my = m.y; d->mog = m.og;
}

__device__ __forceinline__ OffMap lc_load_map(const LcTileDesc *d)
{
    OffMap m;
    m.kind = __ldcg(&d->map_kind); m.v = __ldcg(&d->mv); m.B = __ldcg(&d->mB);
    m.t0 = __ldcg(&d->mt0); m.t1 = __ldcg(&d->mt1); m.y = __ldcg(&d->my); m.og = __ldcg(&d->mog);
    return m;
}

__device__ __forceinline__ OffMap lc_shfl_up_map(const OffMap &m, int off)
{
    OffMap r;
    r.kind = __shfl_up_sync(0xffffffffu, m.kind, off);
    r.v = __shfl_up_sync(0xffffffffu, m.v, off);
    r.B = __shfl_up_sync(0xffffffffu, m.B, off);
    r.t0 = __shfl_up_sync(0xffffffffu, m.t0, off);
    r.t1 = __shfl_up_sync(0xffffffffu, m.t1, off);
    r.y = __shfl_up_sync(0xffffffffu, m.y, off);
    r.og = __shfl_up_sync(0xffffffffu, m.og, off);
    return r;
}

__device__ __forceinline__ unsigned long long lc_gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// neutral element of composition
__device__ __forceinline__ OffMap lc_map_neutral() { return lc_map_trans(0.0, 0.0, 0.0); }

#define LC_CUDA_OK(expr)                                                                   \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) return lc_fail(ctx, _e, #expr, __FILE__, __LINE__);         \
    } while (0)

// ---------------------------------------------------------------------------
// Warp-cooperative decoupled look-back (one full warp).
//
// Tiles publish status 1 + aggregate, later status 2 + inclusive prefix.
// Each round the warp inspects 32 predecessors at once (lane 0 = nearest),
// stops at the nearest inclusive one and folds the aggregates in between
// with a shuffle tree.  op(a, b) means "a then b" (a is the earlier tile).
// st_of(k) must be an acquire load; val_of(k, st) the matching value.
// `first` is the value before tile 0 (the launch state; ident by default).
template <typename T, typename Op, typename Shfl, typename StOf, typename ValOf>
__device__ __forceinline__ T lc_lookback_warp(long long t, T ident, Op op, Shfl shfl_down,
                                             StOf st_of, ValOf val_of, const T *first = nullptr)
{
    const int lane = threadIdx.x & 31;
    T acc = ident;                                // prefix of tiles already folded (later ones)
    long long k = t - 1;
    for (;;) {
        const long long idx = k - lane;
        int st = 2;
        T v = (idx == -1 && first) ? *first : ident;
        if (idx >= 0) {
            while ((st = st_of(idx)) == 0) { }
            v = val_of(idx, st);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, st == 2);
        const int j = incl ? __ffs(incl) - 1 : 32;
        if (lane > j) v = ident;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T other = shfl_down(v, off);
            if (lane + off < 32) v = op(other, v);
        }
        acc = op(v, acc);                         // valid on lane 0
        if (j < 32) break;
        k -= 32;
    }
    return acc;                                   // lane 0 holds the exclusive prefix
}

__device__ __forceinline__ OffMap lc_shfl_down_map(const OffMap &m, int off)
{
    OffMap r;
    r.kind = __shfl_down_sync(0xffffffffu, m.kind, off);
    r.v = __shfl_down_sync(0xffffffffu, m.v, off);
    r.B = __shfl_down_sync(0xffffffffu, m.B, off);
    r.t0 = __shfl_down_sync(0xffffffffu, m.t0, off);
    r.t1 = __shfl_down_sync(0xffffffffu, m.t1, off);
    r.y = __shfl_down_sync(0xffffffffu, m.y, off);
    r.og = __shfl_down_sync(0xffffffffu, m.og, off);
    return r;
}

__device__ __forceinline__ int ld_relaxed(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Block-wide decoupled look-back: all LC_TPB threads inspect LC_TPB
// predecessors per round (thread 0 = nearest), so the inclusive-prefix front
// advances a whole resident wave per round.  Only the tiles nearer than the
// nearest inclusive one are waited for (relaxed polling with back-off, one
// acquire load per used descriptor).  Must be called by every thread of the
// block; returns the exclusive prefix on every thread.
// st_ptr(k): address of tile k's status word; val_of(k, st) its value.
template <typename T, typename Op, typename Shfl, typename StPtr, typename ValOf>
__device__ __forceinline__ T lc_lookback_block(long long t, T ident, Op op, Shfl shfl_down, StPtr st_ptr,
                                              ValOf val_of, T *scratch, int *sj, T *result,
                                              unsigned long long *dbg = nullptr)
// (sj unused; kept for call-site compatibility)
{
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    __shared__ unsigned s_incl[LC_TPB / 32], s_zero[LC_TPB / 32];
    T acc = ident;
    long long k = t - 1;
    for (;;) {
        const long long idx = k - tid;
        int st = idx >= 0 ? 0 : 2;
        int j;
        for (int round = 0;; ++round) {
            if (st == 0) st = ld_relaxed(st_ptr(idx));
            const unsigned incl = __ballot_sync(0xffffffffu, st == 2);
            const unsigned zero = __ballot_sync(0xffffffffu, st == 0);
            if (lane == 0) { s_incl[wid] = incl; s_zero[wid] = zero; }
            __syncthreads();
            // every thread derives the same j / miss from the per-warp masks
            j = LC_TPB;
            bool miss = false;
            for (int w = 0; w < LC_TPB / 32; ++w) {
                const unsigned iw = s_incl[w], zw = s_zero[w];
                const unsigned below = iw ? ((1u << (__ffs(iw) - 1)) - 1u) : 0xffffffffu;
                if (zw & below) miss = true;
                if (iw) { j = w * 32 + __ffs(iw) - 1; break; }
            }
            __syncthreads();                          // masks consumed before the next round
            if (!miss) {
                if (dbg && tid == 0) { dbg[0] = lc_gtimer(); dbg[1] = round; dbg[2] = j; }
                break;
            }
            __nanosleep(round < 4 ? 32 : 256);
        }
        T v = ident;
        if (idx >= 0 && tid <= j) {
            st = ld_acquire(st_ptr(idx));            // orders the value loads after the status
            v = tid == j ? val_of(idx, 2) : val_of(idx, 1);
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T other = shfl_down(v, off);
            if (lane + off < 32) v = op(other, v);
        }
        if (lane == 0) scratch[wid] = v;
        __syncthreads();
        if (tid == 0) {
            T r = scratch[LC_TPB / 32 - 1];
            for (int w = LC_TPB / 32 - 2; w >= 0; --w) r = op(r, scratch[w]);
            acc = op(r, acc);
            *result = acc;
        }
        __syncthreads();
        acc = *result;
        if (dbg && tid == 0) dbg[3] = lc_gtimer();
        if (j < LC_TPB) break;
        k -= LC_TPB;
        __syncthreads();
    }
    return acc;
}

// ---- bulk async copy (TMA engine) global -> shared, completion on an mbarrier
__device__ __forceinline__ void lc_mbar_init(unsigned long long *bar, unsigned count)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: expect `bytes` and start the copy (16-byte aligned, multiple of 16)
__device__ __forceinline__ void lc_bulk_load(void *dst, const void *src, unsigned bytes, unsigned long long *bar)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void lc_mbar_wait(unsigned long long *bar, unsigned phase)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(b), "r"(phase) : "memory");
    } while (!ok);
}

// ---- compacted replay of flagged chunks -------------------------------------
// Chunks whose hot loop flagged possible map events are queued in shared memory
// and replayed by consecutive threads (full warps) instead of by their owners
// (one divergent lane per warp).  replay(q) computes the chunk's map and stores
// it where the owner reads it after this call.  Call from all threads.
// Entry = chunk index in the tile with the binade of its guess start (the
// identity map's grid), its flag mask and the chain value before its first
// flagged step (the replay starts there: earlier steps are not events).
struct LcReplayItem {
    int chg;            // chunk | g0 biased exponent << 8 | (g0 == 0) << 19
    unsigned mask;
    double rs;
};
__device__ __forceinline__ int lc_replay_ch(const LcReplayItem &it) { return it.chg & 0xff; }
// ulp(g0) from the packed binade (lc_ulp only reads the exponent and zero-ness)
__device__ __forceinline__ double lc_replay_ulp(const LcReplayItem &it)
{
    const int be = (it.chg >> 8) & 0x7ff;
    if (it.chg >> 19) return 0.0;
    return lc_ulp(be ? lc_from_bits((int64_t)be << 52) : lc_from_bits(1));
}

template <typename Replay>
__device__ __forceinline__ void lc_tile_replay(bool need, unsigned mask, double g0, double rs, LcReplayItem *q,
                                               int *s_cnt, Replay replay)
{
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, need);
    if (lane == 0) s_cnt[wid] = __popc(b);
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < LC_TPB / 32; ++w) {
        const int cw = s_cnt[w];
        base += w < wid ? cw : 0;
        tot += cw;
    }
    if (need) {
        LcReplayItem it;
        it.chg = tid | (int)(((lc_bits(g0) >> 52) & 0x7ff) << 8) | ((g0 == 0.0) << 19);
        it.mask = mask; it.rs = rs;
        q[base + __popc(b & ((1u << lane) - 1u))] = it;
    }
    __syncthreads();
    for (int k = tid; k < tot; k += LC_TPB) replay(q[k]);
    __syncthreads();
}

// OffMap <-> 14 shared-memory words (rows of 32-bit codes are only 4-byte aligned)
__device__ __forceinline__ void lc_map_to_words(uint32_t *w, const OffMap &m)
{
    const double f[6] = {m.v, m.B, m.t0, m.t1, m.y, m.og};
    w[0] = (uint32_t)m.kind;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        w[1 + 2 * i] = (uint32_t)__double2loint(f[i]);
        w[2 + 2 * i] = (uint32_t)__double2hiint(f[i]);
    }
}

__device__ __forceinline__ OffMap lc_map_from_words(const uint32_t *w)
{
    double f[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) f[i] = __hiloint2double((int)w[2 + 2 * i], (int)w[1 + 2 * i]);
    OffMap m;
    m.kind = (int)w[0];
    m.v = f[0]; m.B = f[1]; m.t0 = f[2]; m.t1 = f[3]; m.y = f[4]; m.og = f[5];
    return m;
}

// ---- asynchronous global -> shared copies (LDGSTS) and L2 prefetch ----------
__device__ __forceinline__ void lc_cp_async8(void *smem_dst, const void *gsrc)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void lc_cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void lc_cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void lc_prefetch_l2(const void *p)
{
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// L2 prefetch of [p, p + bytes) by the whole CTA (one 128-byte line per thread
// and round); used to warm the next tile's inputs while the current one runs.
__device__ __forceinline__ void lc_prefetch_bytes(const void *p, size_t bytes)
{
    const char *c = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)127);
    const char *e = reinterpret_cast<const char *>(p) + bytes;
    for (const char *q = c + 128 * threadIdx.x; q < e; q += 128 * blockDim.x) lc_prefetch_l2(q);
}

__device__ __forceinline__ OffMap lc_shfl_idx_map(const OffMap &m, int src)
{
    OffMap r;
    r.kind = __shfl_sync(0xffffffffu, m.kind, src);
    r.v = __shfl_sync(0xffffffffu, m.v, src);
    r.B = __shfl_sync(0xffffffffu, m.B, src);
    r.t0 = __shfl_sync(0xffffffffu, m.t0, src);
    r.t1 = __shfl_sync(0xffffffffu, m.t1, src);
    r.y = __shfl_sync(0xffffffffu, m.y, src);
    r.og = __shfl_sync(0xffffffffu, m.og, src);
    return r;
}

// Inclusive warp scan of chunk maps (lane 0 earliest), in place.  Call from all
// 32 lanes.  LANE-UNIFORM CONTROL FLOW ONLY: no lane ever runs a composition
// the other lanes do not run.  (The earlier form -- `if (lane >= o) inc =
// compose(inc, up)` per shuffle round -- left a lane split off from its warp
// on sm_100a after a long composition on config 4's 256^3 GMRES vector: ptxas
// had removed the warp barriers it believed redundant, the next shuffles read
// inactive lanes, and pass A's tile loop never ended for the lone lane.)
//   1. every lane a translation with a non-zero grid (chunks without events):
//      prefix sum of y, lane 0's grid fields;
//   2. translations and constants only (constants: chunks with an escape):
//      the same shuffle rounds with the composition written as selects;
//   3. otherwise (a periodic or invalid map somewhere): 32 sequential
//      compositions on broadcast operands, identical in every lane.
// Compositions are exact (power-of-two grids), so the order does not matter.
__device__ __forceinline__ void lc_warp_scan_maps(OffMap &inc)
{
    const int lane = threadIdx.x & 31;
    if (__all_sync(0xffffffffu, inc.kind == LC_MAP_TRANS && inc.v != 0.0)) {
        double y = inc.y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double up = __shfl_up_sync(0xffffffffu, y, o);
            y = lane >= o ? up + y : y;
        }
        inc.y = y;
        inc.v = __shfl_sync(0xffffffffu, inc.v, 0);
        inc.B = __shfl_sync(0xffffffffu, inc.B, 0);
        inc.t0 = __shfl_sync(0xffffffffu, inc.t0, 0);
        inc.t1 = __shfl_sync(0xffffffffu, inc.t1, 0);
        inc.og = __shfl_sync(0xffffffffu, inc.og, 0);
        return;
    }
    if (__all_sync(0xffffffffu, inc.kind == LC_MAP_TRANS || inc.kind == LC_MAP_CONST)) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const OffMap up = lc_shfl_up_map(inc, o);
            // lc_map_compose(inc, up) for these kinds: a constant `inc` absorbs `up`; a
            // constant `up` gives the constant up.y + inc.y; two translations add, the
            // grid fields come from `up` unless it is the neutral map (v == 0)
            const bool use = lane >= o && inc.kind != LC_MAP_CONST;
            const bool upc = up.kind == LC_MAP_CONST;
            const bool own = !upc && up.v == 0.0;
            const double y = up.y + inc.y;
            inc.kind = use ? (upc ? (int)LC_MAP_CONST : (int)LC_MAP_TRANS) : inc.kind;
            inc.y = use ? y : inc.y;
            inc.v = use ? (upc ? 0.0 : (own ? inc.v : up.v)) : inc.v;
            inc.B = use ? (upc ? 0.0 : (own ? inc.B : up.B)) : inc.B;
            inc.t1 = use ? (upc ? 0.0 : (own ? inc.t1 : up.t1)) : inc.t1;
            inc.og = use ? (upc ? 0.0 : (own ? inc.og : up.og)) : inc.og;
            inc.t0 = use ? (upc ? 0.0 : up.t0) : inc.t0;
        }
        return;
    }
    const OffMap mine = inc;
    OffMap acc = lc_map_neutral();
    for (int l = 0; l < 32; ++l) {
        const OffMap m = lc_shfl_idx_map(mine, l);
        acc = lc_map_compose(m, acc);                // the same operands in every lane
        const bool me = lane == l;
        inc.kind = me ? acc.kind : inc.kind;
        inc.v = me ? acc.v : inc.v;
        inc.B = me ? acc.B : inc.B;
        inc.t0 = me ? acc.t0 : inc.t0;
        inc.t1 = me ? acc.t1 : inc.t1;
        inc.y = me ? acc.y : inc.y;
        inc.og = me ? acc.og : inc.og;
    }
}

// Inclusive scan (in place) of nw <= 32 per-warp map aggregates by warp 0; call
// from all threads between two __syncthreads().
__device__ __forceinline__ void lc_scan_warp_maps(OffMap *agg, int nw)
{
    if ((threadIdx.x >> 5) == 0) {
        const int lane = threadIdx.x & 31;
        OffMap v = lane < nw ? agg[lane] : lc_map_neutral();
        lc_warp_scan_maps(v);
        if (lane < nw) agg[lane] = v;
    }
}
