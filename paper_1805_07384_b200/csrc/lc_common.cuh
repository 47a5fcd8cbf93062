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

// neutral element of composition
__device__ __forceinline__ OffMap lc_map_neutral() { return lc_map_trans(0.0, 0.0, 0.0); }

#define LC_CUDA_OK(expr)                                                                   \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) return lc_fail(ctx, _e, #expr, __FILE__, __LINE__);         \
    } while (0)
