// lc_decode.cu -- chunk-parallel canonical Huffman decode and exact-chain
// reconstruction (sm_100a).
//
// Replaces huffman.decode/_decode_tables/_decode_kernel (huffman.py:75-93,
// 110-132, 153-172) and _decompress_kernel + the escape checks of
// compressor.decompress (compressor.py:358-376, 420-440).
//
// Huffman decode of a v1 (LCKP0001) bitstream, which has no sync points:
//   * the bitstream is cut into 128-bit segments, one thread each, 256
//     consecutive segments per CTA;
//   * every segment first decodes from its own base; a segment records the
//     positions of its codeword starts as a 128-bit mask.  Re-decoding from a
//     corrected start stops at the first start shared with the previous walk
//     (from there both walks coincide), so corrections are cheap;
//   * corrections are propagated inside the CTA in shared memory until no
//     exit moves, then across CTAs by short host-driven passes (canonical
//     codes resynchronise within a few codewords, so one pass is typical);
//   * counts are scanned to output offsets and a final pass writes symbols;
//     a 12-bit table yields every codeword that fits in the next 12 bits;
//   * the first decoding anomaly on the true path reproduces the reference
//     status (1 invalid codeword, 2 exhausted, 3 trailing bits).
// Reconstruction runs the same chunked exact chain as the encoder
// (lc_chain.cuh): guesses from the m-prefix since the last escape, offset
// maps + look-back, exact re-run, end/start checks (host relaunch on failure).
#include <type_traits>
#include <cub/block/block_scan.cuh>
#include "lc_kernels.cuh"
#include "../../include/lossyckpt_b200.h"

#define LC_LUT_BITS 12
#define LC_DEC_TPB 256
#define LC_SEG_DEAD 0xffffu
#define LC_L16 4096                  // second-level length table (16-bit prefixes of long codes)

struct LcDecTables {
    int max_len;
    int used;
    int status;                      // 0 ok, 1 unsupported (max_len > 64)
    int pad;
    unsigned long long first_code[66];
    unsigned long long count[66];
    unsigned long long offset[66];
    unsigned int lut[1 << LC_LUT_BITS];   // (len << 24) | sym; ~0 = no code of length <= LUT_BITS
    unsigned int lut2[1 << LC_LUT_BITS];  // codewords inside the 12 bits: (n << 16) | (bits << 12) | start mask
    unsigned long long lim[34];      // left-justified 32-bit code limits per length (canonical codes, l <= 32)
    int canon;                       // Kraft <= 1 and max_len <= 32: lengths follow from lim[]
    unsigned s16;                    // first 16-bit prefix of the codes longer than LC_LUT_BITS (canonical)
    int pad2[2];
    unsigned char len16[LC_L16];     // length (13..16) of the code under 16-bit prefix s16 + i; 0: longer / none
};

// The part of LcDecTables the segment sync walk reads (multi-codeword LUT and
// long-code lengths): ~21 KB of shared memory instead of ~39 KB, so more sync
// CTAs fit per SM.  Rare slow paths read the full table from global memory.
struct LcDecSyncTables {
    int max_len;
    int canon;
    unsigned s16;
    int pad;
    unsigned long long lim[34];
    unsigned int lut2[1 << LC_LUT_BITS];
    unsigned char len16[LC_L16];
};

// lengths[nl] -> tables + sorted symbols (canonical order).  SM: the lengths
// are first staged in shared memory with 16-byte loads (nl <= LC_DEC_LEN_SMEM).
#define LC_DEC_LEN_SMEM 98304
template <bool SM>
__global__ void __launch_bounds__(1024) lc_dec_tables_kernel(const uint8_t *__restrict__ glengths, uint32_t nl,
                                                            LcDecTables *__restrict__ T,
                                                            uint32_t *__restrict__ sorted)
{
    extern __shared__ __align__(16) uint8_t s_lengths[];
    if (SM) {
        const uint32_t nv = (nl + 15) / 16;
        const bool al = (reinterpret_cast<uintptr_t>(glengths) & 15) == 0;
        for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
            uint4 v;
            if (al && 16 * i + 16 <= nl) {
                v = __ldg(reinterpret_cast<const uint4 *>(glengths) + i);
            } else {
                uint8_t b[16];
                for (int k = 0; k < 16; ++k) b[k] = 16 * i + k < nl ? glengths[16 * i + k] : 0;
                v = *reinterpret_cast<uint4 *>(b);
            }
            reinterpret_cast<uint4 *>(s_lengths)[i] = v;
        }
    }
    const uint8_t *lengths = SM ? s_lengths : glengths;
    __shared__ int s_cnt[66];
    __shared__ int s_wcnt[32][66];
    __shared__ int s_max;
    __shared__ unsigned long long s_first[66], s_off[66];
    __shared__ unsigned int s_lut[1 << LC_LUT_BITS];
    __shared__ unsigned long long s_lim[34];         // T->lim, kept on chip for the length table below
    __shared__ unsigned s_s16;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    if (tid < 66) s_cnt[tid] = 0;
    if (tid == 0) s_max = 0;
    for (int i = tid; i < 32 * 66; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t span = (nl + nw - 1) / nw;
    const uint32_t sb = wid * span, se = min(nl, sb + span);
    for (uint32_t s0 = sb; s0 < se; s0 += 32) {
        const uint32_t s = s0 + lane;
        const int l = s < se ? lengths[s] : 0;
        if (l > 0) {
            atomicMax(&s_max, l);
            if (l <= 64) { atomicAdd(&s_wcnt[wid][l], 1); atomicAdd(&s_cnt[l], 1); }
        }
    }
    __syncthreads();
    if (tid == 0) {
        // huffman.py:86-90 (first_code / offsets per length)
        unsigned long long code = 0, off = 0;
        const int ml = s_max;
        int used = 0;
        for (int l = 1; l <= 64; ++l) {
            s_first[l] = code;
            s_off[l] = off;
            T->first_code[l] = code;
            T->count[l] = s_cnt[l];
            T->offset[l] = off;
            code = (code + s_cnt[l]) << 1;
            off += s_cnt[l];
            used += s_cnt[l];
        }
        T->max_len = ml;
        T->used = used;
        T->status = ml > 64 ? 1 : 0;
        // canonical ranges are contiguous and ordered by length when no
        // length overflows its code space (Kraft <= 1)
        int canon = ml <= 32;
        for (int l = 1; l <= 32; ++l)
            if (s_first[l] + (unsigned long long)s_cnt[l] > (1ULL << l)) canon = 0;
        for (int l = 0; l <= 33; ++l) {
            unsigned long long v = ~0ULL;
            if (canon && l >= 1 && l <= 32 && l < ml)
                v = (s_first[l] + (unsigned long long)s_cnt[l]) << (32 - l);
            else if (canon && l == ml)
                v = (s_first[l] + (unsigned long long)s_cnt[l]) << (32 - l);
            T->lim[l] = v;
            s_lim[l] = v;
        }
        T->canon = canon;
        // long canonical codes occupy the 12-bit prefixes from lim[12] upwards
        s_s16 = (canon && ml > LC_LUT_BITS) ? (unsigned)(s_lim[LC_LUT_BITS] >> 16) : 0x10000u;
        T->s16 = s_s16;
    }
    __syncthreads();
    {
        // lengths 13..16 depend on the top 16 bits only (lim[l] is a multiple
        // of 2^16 for l <= 16); same rule as lc_long_len.  (Limits read from shared memory:
        // reading T->lim back from global memory put ~10 dependent L2 round trips here.)
        const unsigned s16 = s_s16;
        const int ml = s_max;
        for (int i = tid; i < LC_L16; i += blockDim.x) {
            const unsigned w16 = s16 + (unsigned)i;
            int len = 0;
            if (w16 < 0x10000u) {
                const unsigned long long w = (unsigned long long)w16 << 16;
                if (w < s_lim[ml <= 32 ? ml : 32])
                    for (int l = LC_LUT_BITS + 1; l <= 16 && l <= ml; ++l)
                        if (w < s_lim[l]) { len = l; break; }
            }
            T->len16[i] = (unsigned char)len;
        }
    }
    if (tid >= 1 && tid <= 64 && s_cnt[tid]) {
        int acc = 0;
        for (int w = 0; w < nw; ++w) {
            const int c0 = s_wcnt[w][tid];
            s_wcnt[w][tid] = acc;
            acc += c0;
        }
    }
    __syncthreads();
    for (uint32_t s0 = sb; s0 < se; s0 += 32) {
        const uint32_t s = s0 + lane;
        const int l = s < se ? lengths[s] : 0;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        if (l > 0 && l <= 64) {
            const int rank = s_wcnt[wid][l] + __popc(peers & ((1u << lane) - 1u));
            sorted[s_off[l] + rank] = s;
        }
        __syncwarp();
        if (l > 0 && l <= 64 && (int)(__ffs(peers) - 1) == lane) s_wcnt[wid][l] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // single-codeword table: the reference tries lengths in increasing order
    // (huffman.py:117-125), so the shortest matching length wins; codes that
    // overflow their length never match
    for (int w = tid; w < (1 << LC_LUT_BITS); w += blockDim.x) {
        unsigned e = 0xffffffffu;
        for (int l = 1; l <= LC_LUT_BITS; ++l) {
            const unsigned long long v = (unsigned long long)(w >> (LC_LUT_BITS - l));
            const unsigned long long rel = v - s_first[l];
            if (s_cnt[l] && v >= s_first[l] && rel < (unsigned long long)s_cnt[l]) {
                e = ((unsigned)l << 24) | sorted[s_off[l] + rel];
                break;
            }
        }
        s_lut[w] = e;
    }
    __syncthreads();
    // Multi-codeword entries.  A codeword found with padded (unknown) low bits
    // is exact when it ends inside the known bits: every shorter codeword
    // depends on known bits only, and the table keeps the shortest match.
    for (int w = tid; w < (1 << LC_LUT_BITS); w += blockDim.x) {
        const unsigned e0 = s_lut[w];
        T->lut[w] = e0;
        unsigned sm = 0;
        int pos = 0, n = 0;
        while (pos < LC_LUT_BITS) {
            const unsigned e = s_lut[(w << pos) & ((1 << LC_LUT_BITS) - 1)];
            if (e == 0xffffffffu) break;
            const int l = (int)(e >> 24);
            if (pos + l > LC_LUT_BITS) break;
            sm |= 1u << pos;
            pos += l;
            ++n;
        }
        T->lut2[w] = n ? ((unsigned)n << 16) | ((unsigned)pos << 12) | sm : 0u;
    }
}

// Decode one codeword at bit p.  Returns its length (>0) and *sym, or 0 for
// "no codeword within max_len bits".
__device__ __forceinline__ int lc_decode_one(const LcDecTables &T, const uint32_t *__restrict__ sorted,
                                             unsigned long long win, int max_len, uint32_t *sym)
{
    const uint32_t e = T.lut[win >> (64 - LC_LUT_BITS)];
    if (e != 0xffffffffu) { *sym = e & 0xffffffu; return (int)(e >> 24); }
    for (int l = LC_LUT_BITS + 1; l <= max_len; ++l) {
        const unsigned long long v = win >> (64 - l);
        const unsigned long long rel = v - T.first_code[l];
        if (v >= T.first_code[l] && rel < T.count[l]) { *sym = sorted[T.offset[l] + rel]; return l; }
    }
    return 0;
}

// Per-segment decode state (8 bytes).  Positions are relative to the
// segment base; `start` == LC_SEG_DEAD: the decode path ended before it.
struct __align__(8) LcSeg {
    unsigned short start;        // first codeword start
    unsigned short exit;         // first codeword start >= segment end, or stop point
    unsigned short count;        // codewords started in [start, exit)
    unsigned char term;          // 0 none, 1 invalid, 2 exhausted, 4 clean end at bit_length, 8 dead
    unsigned char pad;
};

struct LcBlkOut {                // exit of a CTA's last segment (absolute; ~0 when it terminated)
    unsigned long long exit;
};

struct LcDecParams {
    const uint32_t *payload;    // words (big-endian bit order inside bytes), padded
    unsigned long long bits;    // bit_length
    const LcDecTables *T;
    const uint32_t *sorted;
    unsigned long long nseg;
    long long nblk;             // CTAs of LC_DEC_TPB segments
    int seg_bits;               // 64 * sub-segments
    unsigned long long nwords;  // payload words readable (padded)
};

// staged words beyond a CTA's segments: the last walk reads at most one
// codeword (<= 64 bits) past its segment plus the reader's 64-bit lookahead
#define LC_DEC_STAGE_PAD 8
#define LC_DEAD32 0xffffffffu

static size_t lc_dec_stage_bytes(int ns)
{
    return sizeof(uint32_t) * (LC_DEC_TPB * 2 * ns + LC_DEC_STAGE_PAD) + 8ull * LC_DEC_TPB * ns;
}

// Payload word sources for the bit reader (32-bit word index relative to a
// base the caller chose): global memory, or a CTA range staged in shared
// memory.  Words are big-endian byte streams.
struct LcGlobSrc {
    const uint32_t *w;
    __device__ __forceinline__ uint32_t word(unsigned i) const { return __byte_perm(__ldg(w + i), 0, 0x0123); }
};
struct LcSmemSrc {
    const uint32_t *w;
    __device__ __forceinline__ uint32_t word(unsigned i) const { return __byte_perm(w[i], 0, 0x0123); }
};

// MSB-first bit reader over relative bit positions: the top nb bits of buf
// are valid (nb in (32, 64] after refill).
template <class Src>
struct LcBitReader {
    Src src;
    unsigned long long buf;
    unsigned pos, next;
    int nb;
    __device__ __forceinline__ void seek(unsigned p)
    {
        pos = p;
        const unsigned wi = p >> 5;
        const int sh = (int)(p & 31);
        buf = (((unsigned long long)src.word(wi) << 32) | src.word(wi + 1)) << sh;
        nb = 64 - sh;
        next = wi + 2;
        if (nb <= 32) refill();
    }
    __device__ __forceinline__ void refill()
    {
        buf |= (unsigned long long)src.word(next) << (32 - nb);
        ++next;
        nb += 32;
    }
    __device__ __forceinline__ void consume(int l)
    {
        if (l >= nb) { seek(pos + l); return; }      // only for codes longer than the buffer
        buf <<= l;
        nb -= l;
        pos += l;
        if (nb <= 32) refill();
    }
    // 64 bits from pos (for codes longer than the buffered bits)
    __device__ __forceinline__ unsigned long long window(int max_len) const
    {
        if (max_len <= nb) return buf;
        const unsigned wi = pos >> 5;
        const int sh = (int)(pos & 31);
        const unsigned long long hi = ((unsigned long long)src.word(wi) << 32) | src.word(wi + 1);
        if (!sh) return hi;
        return (hi << sh) | ((unsigned long long)src.word(wi + 2) >> (32 - sh));
    }
};

// bit_length relative to a base bit (clamped; 0 when the stream ended before it)
__device__ __forceinline__ unsigned lc_bits_rel(unsigned long long bits, unsigned long long base)
{
    if (bits <= base) return 0u;
    const unsigned long long r = bits - base;
    return r > 0x7fffffffull ? 0x7fffffffu : (unsigned)r;
}

// One codeword at the reader; returns its length, 0 for "no codeword within
// max_len bits"; sets *term for anomalies exactly like huffman.py:114-129.
template <class BR>
__device__ __forceinline__ int lc_next_symbol(const LcDecTables &T, const uint32_t *__restrict__ sorted,
                                              const BR &br, unsigned bits_rel, uint32_t *sym, int *term)
{
    if (br.pos >= bits_rel) { *term = 4; return 0; }
    const unsigned remaining = bits_rel - br.pos;
    const int max_len = T.max_len;
    const int l = lc_decode_one(T, sorted, br.window(max_len), max_len, sym);
    if (l == 0) { *term = remaining > (unsigned)max_len ? 1 : 2; return 0; }
    if ((unsigned)l > remaining) { *term = 2; return 0; }
    return l;
}

// Length of a codeword longer than LC_LUT_BITS for canonical codes (T.canon):
// the first length whose left-justified limit exceeds the window.  Returns 0
// when the window is past every code (the exact path then decides).
template <class TT>
__device__ __forceinline__ int lc_long_len(const TT &T, unsigned long long buf)
{
    const unsigned long long w = buf >> 32;
    if (!T.canon || w >= T.lim[T.max_len]) return 0;
    int l = LC_LUT_BITS + 1;                 // long codes are rare and mostly just over 12 bits
#pragma unroll 1
    while (w >= T.lim[l]) ++l;
    return l;
}

// lc_long_len through the 16-bit second-level table (codes of 13..16 bits),
// the limit walk for longer ones
template <class TT>
__device__ __forceinline__ int lc_long_len_fast(const TT &T, unsigned long long buf)
{
    const unsigned i = (unsigned)(buf >> 48) - T.s16;
    const int l = i < (unsigned)LC_L16 ? (int)T.len16[i] : 0;
    return l ? l : lc_long_len(T, buf);
}

__device__ __forceinline__ void lc_seg_dead(LcSeg &S)
{
    S.start = S.exit = LC_SEG_DEAD;
    S.count = 0;
    S.term = 8;
}

// Walk codewords from `start` (CTA-relative bit) until the first codeword
// start >= segment end (the exit) or an anomaly.  The segment is NS
// sub-segments of 64 bits; Ms[k * LC_DEC_TPB] (shared memory, conflict-free
// across the warp) holds the codeword-start mask of sub-segment k: the
// previous walk's when `resync`, replaced by this one's.  With `resync` the
// walk stops at the first start both walks share: from there on they
// coincide (count, exit and status carry over).
template <int NS>
__device__ void lc_seg_walk(const LcDecSyncTables &T, const LcDecTables &Tg, const uint32_t *__restrict__ sorted,
                            const LcSmemSrc &src,
                            unsigned bits_rel, unsigned seg_rel, unsigned start, bool resync, LcSeg &S,
                            unsigned long long *Ms)
{
    LcBitReader<LcSmemSrc> br;
    br.src = src;
    br.seek(start);
    int cnt = 0, term = 0, k = 0;
    bool merged = false, stopped = false;
    for (; k < NS; ++k) {
        const unsigned sub_base = seg_rel + 64u * k, sub_end = sub_base + 64u;
        unsigned long long *mw = Ms + k * LC_DEC_TPB;
        const unsigned long long old = resync ? *mw : 0ull;
        unsigned long long mask = 0;
        while (br.pos < sub_end) {
            if (br.pos >= bits_rel) { term = 4; stopped = true; break; }
            const unsigned e2 = T.lut2[br.buf >> (64 - LC_LUT_BITS)];
            int adv = (int)((e2 >> 12) & 15u);
            unsigned sm = e2 & 0xfffu;
            if (!e2 || br.pos + (unsigned)adv > bits_rel) {
                adv = e2 ? 0 : lc_long_len_fast(T, br.buf);
                if (!adv || br.pos + (unsigned)adv > bits_rel) {
                    uint32_t sym;
                    adv = lc_next_symbol(Tg, sorted, br, bits_rel, &sym, &term);
                    if (!adv) { stopped = true; break; }
                }
                sm = 1u;
            }
            const unsigned lim = sub_end - br.pos;
            const unsigned inside = lim >= LC_LUT_BITS ? sm : (sm & ((1u << lim) - 1u));
            const unsigned long long news = (unsigned long long)inside << (br.pos - sub_base);
            const unsigned long long hit = news & old;
            if (hit) {                                   // synchronised with the previous walk
                const unsigned long long below = (hit & (~hit + 1ull)) - 1ull;
                mask = mask | (news & below) | (old & ~below);
                merged = true;
                break;
            }
            mask |= news;
            const unsigned beyond = sm ^ inside;
            if (beyond) { br.consume(__ffs(beyond) - 1); break; }
            br.consume(adv);
        }
        cnt += __popcll(mask);
        *mw = mask;
        if (merged || stopped) break;
    }
    for (int j = k + 1; j < NS; ++j) {
        unsigned long long *mw = Ms + j * LC_DEC_TPB;
        if (merged) cnt += __popcll(*mw);             // old starts carry over
        else *mw = 0ull;
    }
    S.count = (unsigned short)cnt;
    S.start = (unsigned short)(start - seg_rel);
    if (!merged) {
        S.exit = (unsigned short)(br.pos - seg_rel);
        S.term = (unsigned char)term;
    }
}

__device__ __forceinline__ void lc_load_sync_tables(LcDecSyncTables &Ts, const LcDecTables *T)
{
    if (threadIdx.x == 0) { Ts.max_len = T->max_len; Ts.canon = T->canon; Ts.s16 = T->s16; }
    for (int i = threadIdx.x; i < 34; i += blockDim.x) Ts.lim[i] = T->lim[i];
    for (int i = threadIdx.x; i < (1 << LC_LUT_BITS) / 4; i += blockDim.x)
        reinterpret_cast<uint4 *>(Ts.lut2)[i] = __ldg(reinterpret_cast<const uint4 *>(T->lut2) + i);
    for (int i = threadIdx.x; i < LC_L16 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(Ts.len16)[i] = __ldg(reinterpret_cast<const uint4 *>(T->len16) + i);
    __syncthreads();
}

__device__ __forceinline__ void lc_load_tables(LcDecTables &Ts, const LcDecTables *T)
{
    for (int i = threadIdx.x; i < (int)(sizeof(LcDecTables) / 16); i += blockDim.x)
        reinterpret_cast<uint4 *>(&Ts)[i] = __ldg(reinterpret_cast<const uint4 *>(T) + i);
    __syncthreads();
}

// One sync pass.  First pass: every segment walks from its own base, then
// exits are propagated inside each CTA until nothing moves (re-walks stop at
// the first codeword start shared with the previous walk).  Later passes: a
// CTA whose entry (the previous CTA's exit from the last pass) differs from
// its first segment's start re-walks from it and propagates again; *changed
// is set when a CTA's own exit moves (the next CTA then needs another pass).
// The CTA's payload range is staged in shared memory by one bulk copy and
// all positions are 32-bit, relative to the CTA's first bit.
template <int NS>
__global__ void __launch_bounds__(LC_DEC_TPB) lc_dec_sync_kernel(LcDecParams P, LcSeg *__restrict__ seg,
                                                                const LcBlkOut *__restrict__ bprev,
                                                                LcBlkOut *__restrict__ bcur, int first_pass,
                                                                int *__restrict__ changed, const int *need)
{
    if (need && *(volatile const int *)need == 0) return;   // speculative general pass not needed
    __shared__ LcDecSyncTables Ts;
    __shared__ unsigned s_exit[LC_DEC_TPB];
    __shared__ int s_skip;
    __shared__ unsigned long long s_bar;
    extern __shared__ __align__(16) uint32_t s_words[];   // lc_dec_stage_bytes(NS): payload, then masks
    constexpr int NW = LC_DEC_TPB * 2 * NS + LC_DEC_STAGE_PAD;
    constexpr unsigned SEGB = 64u * NS;
    if (threadIdx.x == 0) lc_mbar_init(&s_bar, 1);
    unsigned phase = 0;
    lc_load_sync_tables(Ts, P.T);
    const int tid = threadIdx.x;
    unsigned long long *M = reinterpret_cast<unsigned long long *>(s_words + NW) + tid;
    LcSmemSrc src;
    src.w = s_words;
    const unsigned seg_rel = tid * SEGB;
    for (long long b = blockIdx.x; b < P.nblk; b += gridDim.x) {
        const unsigned long long t = (unsigned long long)b * LC_DEC_TPB + tid;
        const bool live = t < P.nseg;
        const unsigned long long cbit = (unsigned long long)b * LC_DEC_TPB * SEGB;
        const unsigned bits_rel = lc_bits_rel(P.bits, cbit);
        LcSeg S;
        bool have_mask = false;
        unsigned my_start = seg_rel, entry = 0u;
        if (!first_pass) {
            if (live) {
                S = seg[t];
                my_start = S.start == LC_SEG_DEAD ? LC_DEAD32 : seg_rel + S.start;
            }
            if (tid == 0) {
                const unsigned long long ex = b > 0 ? bprev[b - 1].exit : 0ull;
                entry = ex == ~0ull ? LC_DEAD32 : (unsigned)(ex - cbit);
                s_skip = entry == my_start;
            }
            __syncthreads();
            const int skip = s_skip;
            if (skip) {
                __syncthreads();
                if (tid == 0) bcur[b] = bprev[b];
                continue;
            }
        }
        // stage this CTA's payload range (+ lookahead) with one bulk copy; the
        // payload buffer is padded to whole CTA ranges
        if (tid == 0) lc_bulk_load(s_words, P.payload + cbit / 32, (unsigned)(NW * 4), &s_bar);
        lc_mbar_wait(&s_bar, phase);
        phase ^= 1u;
        if (first_pass && live) {
            lc_seg_walk<NS>(Ts, *P.T, P.sorted, src, bits_rel, seg_rel, seg_rel, false, S, M);
            have_mask = true;
        }
        for (;;) {
            s_exit[tid] = (live && !S.term) ? seg_rel + S.exit : LC_DEAD32;
            __syncthreads();
            const unsigned want = tid == 0 ? (first_pass ? 0u : entry) : s_exit[tid - 1];
            bool ch = false;
            if (live && want != my_start) {
                if (want == LC_DEAD32) { lc_seg_dead(S); have_mask = false; }
                else { lc_seg_walk<NS>(Ts, *P.T, P.sorted, src, bits_rel, seg_rel, want, have_mask, S, M); have_mask = true; }
                my_start = want;
                ch = true;
            }
            if (!__syncthreads_or(ch)) break;
        }
        if (live) seg[t] = S;
        if (tid == LC_DEC_TPB - 1) {
            const unsigned long long ex = (live && !S.term) ? cbit + seg_rel + S.exit : ~0ull;
            bcur[b].exit = ex;
            if (!first_pass && ex != bprev[b].exit) atomicExch(changed, 1);
        }
    }
}

// Boundary fix after the first sync pass: CTA b's first segment was walked
// from its own base, but the true entry is CTA b-1's exit.  One thread per
// CTA boundary re-walks that segment from the entry (payload read through
// L1/L2).  When the new walk reaches the same exit and status, only the
// segment's start and count change and the CTA is final; otherwise the
// exit moved, nothing is written and *changed asks the host for the general
// propagation passes (lc_dec_sync_kernel).
__global__ void __launch_bounds__(128) lc_dec_fix_kernel(LcDecParams P, LcSeg *__restrict__ seg,
                                                         const LcBlkOut *__restrict__ bout, int *__restrict__ changed)
{
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (b >= P.nblk) return;
    const unsigned long long t = (unsigned long long)b * LC_DEC_TPB;
    if (t >= P.nseg) return;
    const unsigned segb = (unsigned)P.seg_bits;
    const unsigned long long sbit = t * segb;
    const unsigned long long ex = bout[b - 1].exit;
    LcSeg S = seg[t];
    const unsigned long long cur = S.start == LC_SEG_DEAD ? ~0ull : sbit + S.start;
    if (ex == cur) return;
    if (ex == ~0ull) { atomicExch(changed, 1); return; }    // the path ended before this CTA
    const LcDecTables &T = *P.T;
    const unsigned bits_rel = lc_bits_rel(P.bits, sbit);
    LcBitReader<LcGlobSrc> br;
    br.src.w = P.payload + sbit / 32;
    br.seek((unsigned)(ex - sbit));
    int cnt = 0, term = 0;
    while (br.pos < segb) {
        if (br.pos >= bits_rel) { term = 4; break; }
        const unsigned e2 = T.lut2[br.buf >> (64 - LC_LUT_BITS)];
        int adv = (int)((e2 >> 12) & 15u);
        unsigned sm = e2 & 0xfffu;
        if (!e2 || br.pos + (unsigned)adv > bits_rel) {
            adv = e2 ? 0 : lc_long_len_fast(T, br.buf);
            if (!adv || br.pos + (unsigned)adv > bits_rel) {
                uint32_t sym;
                adv = lc_next_symbol(T, P.sorted, br, bits_rel, &sym, &term);
                if (!adv) break;
            }
            sm = 1u;
        }
        const unsigned lim = segb - br.pos;
        const unsigned inside = lim >= LC_LUT_BITS ? sm : (sm & ((1u << lim) - 1u));
        cnt += __popc(inside);
        const unsigned beyond = sm ^ inside;
        if (beyond) { br.consume(__ffs(beyond) - 1); break; }
        br.consume(adv);
    }
    if (br.pos != S.exit || term != S.term) { atomicExch(changed, 1); return; }
    S.start = (unsigned short)(ex - sbit);
    S.count = (unsigned short)cnt;
    seg[t] = S;
}

// Device-wide exclusive scan of segment counts (decoupled look-back) and the
// first anomaly on the decode path.
struct LcScanDesc { int st; int pad; unsigned long long agg, incl; };

__global__ void __launch_bounds__(LC_TPB) lc_dec_scan_kernel(const LcSeg *__restrict__ seg, unsigned long long nseg,
                                                            unsigned long long *__restrict__ off,
                                                            LcScanDesc *__restrict__ desc,
                                                            unsigned int *__restrict__ tile_counter,
                                                            unsigned long long *__restrict__ total_and_term)
{
    typedef cub::BlockScan<unsigned long long, LC_TPB> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long sh_tile;
    __shared__ unsigned long long lb_u[LC_TPB / 32], lb_res, sh_in;
    __shared__ int sh_j;
    const int tid = threadIdx.x;
    const int IPT = 8;
    for (;;) {
        __syncthreads();
        if (tid == 0) sh_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const long long t = sh_tile;
        const unsigned long long base = (unsigned long long)t * LC_TPB * IPT;
        if (base >= nseg) break;
        unsigned long long c[IPT], sum = 0;
        for (int k = 0; k < IPT; ++k) {
            const unsigned long long i = base + (unsigned long long)tid * IPT + k;
            c[k] = 0;
            if (i < nseg) {
                const LcSeg S = seg[i];
                c[k] = S.count;
                if (S.term && S.term != 8) atomicMin(&total_and_term[1], i);
            }
            sum += c[k];
        }
        unsigned long long ex, agg;
        Scan(tmp).ExclusiveSum(sum, ex, agg);
        unsigned long long in = 0;
        if (t > 0) {
            if (tid == 0) { __stcg(&desc[t].agg, agg); st_release(&desc[t].st, 1); }
            in = lc_lookback_block<unsigned long long>(
                t, 0ULL, [](unsigned long long a, unsigned long long b) { return a + b; },
                [](unsigned long long v, int o) { return __shfl_down_sync(0xffffffffu, v, o); },
                [&](long long k) { return &desc[k].st; },
                [&](long long k, int st) { return st == 2 ? __ldcg(&desc[k].incl) : __ldcg(&desc[k].agg); },
                lb_u, &sh_j, &lb_res);
        }
        if (tid == 0) {
            __stcg(&desc[t].incl, in + agg);
            st_release(&desc[t].st, 2);
            sh_in = in;
            if ((base + (unsigned long long)LC_TPB * IPT) >= nseg) total_and_term[0] = in + agg;
        }
        __syncthreads();
        unsigned long long o = sh_in + ex;
        for (int k = 0; k < IPT; ++k) {
            const unsigned long long i = base + (unsigned long long)tid * IPT + k;
            if (i < nseg) off[i] = o;
            o += c[k];
        }
    }
}

// Write pass.  A warp owns 32 consecutive segments, whose symbols form one
// contiguous output range: each lane decodes its segment into a shared-memory
// window of `cap` symbols at its output offset, then the warp copies the
// window to global memory with 16-byte stores.  Ranges longer than the window
// take several rounds (lanes pause at the window end; the <= 11 symbols a
// step spills past it move to the front of the next window).
// words of one warp's padded output window: cap + spill (16) + head (< 8)
// codes, plus one padding word per 32
__host__ __device__ inline int lc_dec_stage_words(int cap, int code_bytes)
{
    const int epw = 4 / code_bytes;
    const int words = (cap + 16 + 8 + epw - 1) / epw + 4;
    return words + words / 32 + 2;
}

template <typename CodeT>
__global__ void __launch_bounds__(LC_DEC_TPB) lc_dec_write_kernel(LcDecParams P, const LcSeg *__restrict__ seg,
                                                                 const unsigned long long *__restrict__ off,
                                                                 void *out, unsigned long long m,
                                                                 unsigned long long *__restrict__ end_pos, int cap)
{
    __shared__ LcDecTables Ts;
    __shared__ unsigned long long s_bar;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    constexpr int EPW = 4 / sizeof(CodeT);              // codes per 32-bit word
    constexpr int VEC = 16 / sizeof(CodeT);             // codes per 16-byte store
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned segb = (unsigned)P.seg_bits;
    const int nw_stage = LC_DEC_TPB * (int)(segb / 32) + LC_DEC_STAGE_PAD;    // payload words per CTA range
    uint32_t *s_words = reinterpret_cast<uint32_t *>(s_dyn);
    // per-warp window, one padding word after every 32 words: the lanes' write
    // streams start ~segment-size apart, which without padding falls on few banks
    const int stage_words = lc_dec_stage_words(cap, (int)sizeof(CodeT));
    uint32_t *stagew = reinterpret_cast<uint32_t *>(s_dyn + (size_t)nw_stage * 4) + (size_t)wid * stage_words;
    CodeT *stage = reinterpret_cast<CodeT *>(stagew);
    CodeT *gout = reinterpret_cast<CodeT *>(out);
    if (tid == 0) lc_mbar_init(&s_bar, 1);
    unsigned phase = 0;
    lc_load_tables(Ts, P.T);
    const int max_len = Ts.max_len;
    LcSmemSrc src;
    src.w = s_words;
    for (long long b = blockIdx.x; b < P.nblk; b += gridDim.x) {
        const unsigned long long cbit = (unsigned long long)b * LC_DEC_TPB * segb;
        if (tid == 0) lc_bulk_load(s_words, P.payload + cbit / 32, (unsigned)(nw_stage * 4), &s_bar);
        const unsigned long long t = (unsigned long long)b * LC_DEC_TPB + tid;
        unsigned long long o = 0;
        unsigned todo = 0;
        LcSeg S0;
        S0.start = LC_SEG_DEAD;
        if (t < P.nseg) {
            S0 = seg[t];
            o = off[t];
            if (S0.start != LC_SEG_DEAD) todo = S0.count;
        }
        if (o >= m) todo = 0;
        else if ((unsigned long long)todo > m - o) todo = (unsigned)(m - o);
        const unsigned bits_rel = lc_bits_rel(P.bits, cbit);
        lc_mbar_wait(&s_bar, phase);
        phase ^= 1u;
        const unsigned long long wlo = __shfl_sync(0xffffffffu, o, 0);
        // warp-relative output slots (a warp covers <= 32 * 1024 symbols)
        unsigned orel = (unsigned)(o - wlo), whi = todo ? orel + todo : 0u;
        whi = __reduce_max_sync(0xffffffffu, whi);
        if (whi) {
            const int a = (int)(wlo & (VEC - 1));
            const bool last = todo && o + todo == m;
            LcBitReader<LcSmemSrc> br;
            br.src = src;
            if (todo) br.seek(tid * segb + S0.start);
            for (unsigned wb = 0; wb < whi; wb += (unsigned)cap) {
                const unsigned wend = wb + (unsigned)cap;
                while (todo && orel < wend) {
                    const unsigned p0 = a + (orel - wb);         // logical window index
                    auto put = [&](int k, uint32_t v) {
                        const unsigned p = p0 + k;
                        stage[p + EPW * (p / (32 * EPW))] = (CodeT)v;
                    };
                    const unsigned w12 = (unsigned)(br.buf >> (64 - LC_LUT_BITS));
                    const unsigned e1 = Ts.lut[w12];
                    const unsigned e2 = Ts.lut2[w12];
                    const unsigned n2 = e2 >> 16;
                    const unsigned L2 = (e2 >> 12) & 15u;
                    const bool fits = br.pos + L2 <= bits_rel;
                    if (n2 >= 2 && n2 <= todo && fits) {
                        // several codewords in the next 12 bits; the first is e1.  All
                        // table reads are issued unconditionally (independent), only the
                        // stores are predicated, so their latencies overlap.
                        put(0, e1 & 0xffffffu);
                        unsigned sm = (e2 & 0xfffu) & ((e2 & 0xfffu) - 1u);
                        uint32_t sy[LC_LUT_BITS - 1];
#pragma unroll
                        for (int k = 0; k < LC_LUT_BITS - 1; ++k) {
                            const int i = __ffs(sm) - 1;           // -1 once exhausted
                            sm &= sm - 1;
                            sy[k] = Ts.lut[(w12 << (i & 15)) & ((1u << LC_LUT_BITS) - 1)];
                        }
#pragma unroll
                        for (int k = 0; k < LC_LUT_BITS - 1; ++k)
                            if (k + 1 < (int)n2) put(k + 1, sy[k] & 0xffffffu);
                        br.consume((int)L2);
                        orel += n2;
                        todo -= n2;
                    } else {
                        uint32_t sym;
                        int l;
                        if (e2 && fits) {                        // one codeword of <= 12 bits
                            sym = e1 & 0xffffffu;
                            l = (int)(e1 >> 24);
                        } else {
                            l = e2 ? 0 : lc_long_len_fast(Ts, br.buf);
                            if (l && br.pos + (unsigned)l <= bits_rel) {
                                const unsigned long long v = (br.buf >> 32) >> (32 - l);
                                sym = __ldg(P.sorted + Ts.offset[l] + (v - Ts.first_code[l]));
                            } else {
                                int term = 0;
                                l = lc_next_symbol(Ts, P.sorted, br, bits_rel, &sym, &term);
                                if (!l) { todo = 0; break; }     // cannot happen on the converged path
                            }
                        }
                        put(0, sym);
                        br.consume(l);
                        ++orel;
                        --todo;
                    }
                    if (last && !todo) *end_pos = cbit + br.pos;
                }
                __syncwarp();
                const unsigned len = whi - wb < (unsigned)cap ? whi - wb : (unsigned)cap;
                const int tot = a + (int)len;                     // logical elements in the window
                CodeT *g = gout + (wlo + wb - a);                 // word aligned
                const int nchunks = (tot + VEC - 1) / VEC;        // 16-byte chunks of the window
                for (int c = lane; c < nchunks; c += 32) {
                    uint32_t v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int w = 4 * c + k;
                        v[k] = stagew[w + (w >> 5)];
                    }
                    if (c * VEC >= a && c * VEC + VEC <= tot) {
                        *reinterpret_cast<uint4 *>(g + c * VEC) = make_uint4(v[0], v[1], v[2], v[3]);
                    } else {
#pragma unroll
                        for (int k = 0; k < VEC; ++k) {
                            const int i = c * VEC + k;
                            if (i >= a && i < tot) g[i] = (CodeT)(v[k / EPW] >> (8 * sizeof(CodeT) * (k % EPW)));
                        }
                    }
                }
                __syncwarp();
                if (len == (unsigned)cap) {                       // spill (< 12 codes) to the front
                    for (int k = lane; k < 16; k += 32) {
                        const unsigned ps = a + cap + k, pd = a + k;
                        stage[pd + EPW * (pd / (32 * EPW))] = stage[ps + EPW * (ps / (32 * EPW))];
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();                                 // payload stage is reused by the next range
    }
}

static size_t lc_dec_write_smem(int cap, int code_bytes, int seg_bits)
{
    return sizeof(uint32_t) * (size_t)(LC_DEC_TPB * (seg_bits / 32) + LC_DEC_STAGE_PAD)
         + sizeof(uint32_t) * (size_t)(LC_DEC_TPB / 32) * lc_dec_stage_words(cap, code_bytes);
}

// v2 blocks: decode from the sync table, no segment synchronisation.  Thread
// j decodes the LC_SYNC_K symbols starting at bit sync[j] (the last group:
// the rest) straight into codes[j*LC_SYNC_K ...] with 16-byte stores, and
// checks that it stops exactly at the next sync point (status 6 otherwise;
// 1/2 for an invalid codeword / exhausted payload).
template <typename CodeT>
__global__ void __launch_bounds__(256) lc_dec_v2_kernel(LcDecParams P, const unsigned long long *__restrict__ sync,
                                                       unsigned long long nsync, void *out_, unsigned long long m,
                                                       int *__restrict__ status)
{
    __shared__ LcDecTables Ts;
    lc_load_tables(Ts, P.T);
    constexpr int VEC = 16 / sizeof(CodeT), HALF = VEC / 2, SH = 8 * sizeof(CodeT);
    CodeT *out = reinterpret_cast<CodeT *>(out_);
    const int max_len = Ts.max_len;
    for (unsigned long long j = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; j < nsync;
         j += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long s0 = sync[j], s1 = j + 1 < nsync ? sync[j + 1] : P.bits;
        const unsigned long long o0 = j * LC_SYNC_K;
        if (s0 > s1 || s1 > P.bits || o0 >= m || (j == 0 && s0 != 0)) { atomicExch(status, 6); continue; }
        unsigned todo = (unsigned)(m - o0 < LC_SYNC_K ? m - o0 : LC_SYNC_K);
        const unsigned long long wbase = s0 & ~31ull;
        const unsigned bits_rel = lc_bits_rel(P.bits, wbase);
        LcBitReader<LcGlobSrc> br;
        br.src.w = P.payload + wbase / 32;
        br.seek((unsigned)(s0 - wbase));
        unsigned long long lo = 0, hi = 0, o = o0;
        int cnt = 0, bad = 0;
        auto put = [&](uint32_t sym) {
            const unsigned long long v = (unsigned long long)(CodeT)sym;
            if (cnt < HALF) lo |= v << (SH * cnt);
            else hi |= v << (SH * (cnt - HALF));
            if (++cnt == VEC) {
                *reinterpret_cast<uint4 *>(out + o) = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32),
                                                                (uint32_t)hi, (uint32_t)(hi >> 32));
                o += VEC;
                lo = hi = 0;
                cnt = 0;
            }
        };
        while (todo) {
            const unsigned w12 = (unsigned)(br.buf >> (64 - LC_LUT_BITS));
            const unsigned e1 = Ts.lut[w12];
            const unsigned e2 = Ts.lut2[w12];
            const unsigned n2 = e2 >> 16;
            const unsigned L2 = (e2 >> 12) & 15u;
            const bool fits = br.pos + L2 <= bits_rel;
            if (n2 >= 2 && n2 <= todo && fits) {
                put(e1 & 0xffffffu);
                unsigned sm = (e2 & 0xfffu) & ((e2 & 0xfffu) - 1u);
#pragma unroll
                for (int k = 1; k < LC_LUT_BITS; ++k) {
                    if ((unsigned)k < n2) {
                        const int i = __ffs(sm) - 1;
                        sm &= sm - 1;
                        put(Ts.lut[(w12 << i) & ((1u << LC_LUT_BITS) - 1)] & 0xffffffu);
                    }
                }
                br.consume((int)L2);
                todo -= n2;
            } else {
                uint32_t sym;
                int l;
                if (e2 && fits) {
                    sym = e1 & 0xffffffu;
                    l = (int)(e1 >> 24);
                } else {
                    l = e2 ? 0 : lc_long_len_fast(Ts, br.buf);
                    if (l && br.pos + (unsigned)l <= bits_rel) {
                        const unsigned long long v = (br.buf >> 32) >> (32 - l);
                        sym = __ldg(P.sorted + Ts.offset[l] + (v - Ts.first_code[l]));
                    } else {
                        int term = 0;
                        l = lc_next_symbol(Ts, P.sorted, br, bits_rel, &sym, &term);
                        if (!l) { bad = term == 4 ? 2 : term; break; }
                    }
                }
                put(sym);
                br.consume(l);
                --todo;
            }
        }
        for (int k = 0; k < cnt; ++k)                   // partial last group
            out[o + k] = (CodeT)((k < HALF ? lo >> (SH * k) : hi >> (SH * (k - HALF))));
        if (bad) atomicExch(status, bad);
        else if (wbase + br.pos != s1) atomicExch(status, 6);
    }
}

// v3 blocks: every LC_SYNC_K-th symbol carries its payload bit offset, the
// exact chain value before it and the escape count before it, so each sync
// interval decodes AND reconstructs on its own -- no segment synchronisation,
// no offset maps, one pass.  Thread = interval: it walks its codewords
// (huffman.py:110-132) and runs the reference chain (compressor.py:358-376)
// from the stored start; the warp's lanes step in lockstep and every 32 steps
// the 32 x 32 values staged in shared memory leave as 32 coalesced 256-byte
// rows.  Checks: each interval ends exactly at the next sync point's bit
// offset, chain value and escape count, the first start is first_value
// (status 6: the table disagrees with the payload); decode statuses 1 / 2 as
// v1; escape codes beyond n_esc and escape positions (flags, like
// compressor.py:435-439).
struct LcDecV3Tables {               // the single-codeword part of LcDecTables (~21 KB)
    int max_len, canon;
    unsigned s16;
    int pad;
    unsigned long long lim[34];
    unsigned long long first_code[66];
    unsigned long long offset[66];
    unsigned int lut[1 << LC_LUT_BITS];
    unsigned char len16[LC_L16];
};
#define LC_V3_TPB 256

struct LcV3Final {
    int status;
    int esc_flags[2];                // [0] more escape codes than values, [1] position mismatch
    int pad;
    long long esc_total;             // escape codes in the block
};

// MSB-first bit reader for the v3 walk with a register prefetch ring: the
// payload words reach registers in aligned 16-byte groups loaded two groups
// (256 bits) ahead of use, so a refill never waits on the memory system (the
// L1 is mostly shared memory here, and each lane walks its own stream).
struct LcV3Reader {
    const uint4 *g4;             // payload as 16-byte groups
    uint4 cur, n1, n2;           // group of word `next`, the two after it
    unsigned long long buf;      // top nb bits valid
    unsigned pos, next;          // bits consumed (relative to the group base); next word to buffer
    int nb;
    __device__ __forceinline__ static uint32_t pick(const uint4 &q, unsigned k)
    {
        const uint32_t lo = (k & 1) ? q.y : q.x, hi = (k & 1) ? q.w : q.z;
        return __byte_perm((k & 2) ? hi : lo, 0, 0x0123);
    }
    __device__ __forceinline__ uint32_t take()
    {
        const uint32_t v = pick(cur, next & 3u);
        ++next;
        if ((next & 3u) == 0) {
            cur = n1;
            n1 = n2;
            n2 = __ldg(g4 + (next >> 2) + 2);
        }
        return v;
    }
    __device__ __forceinline__ void seek(unsigned p)
    {
        pos = p;
        next = p >> 5;
        const unsigned gi = next >> 2;
        cur = __ldg(g4 + gi);
        n1 = __ldg(g4 + gi + 1);
        n2 = __ldg(g4 + gi + 2);
        const int sh = (int)(p & 31);
        const uint32_t w0 = take(), w1 = take();
        buf = (((unsigned long long)w0 << 32) | w1) << sh;
        nb = 64 - sh;
        if (nb <= 32) { buf |= (unsigned long long)take() << (32 - nb); nb += 32; }
    }
    __device__ __forceinline__ void consume(int l)
    {
        if (l >= nb) { seek(pos + l); return; }      // codes longer than the buffer (rare)
        buf <<= l;
        nb -= l;
        pos += l;
        if (nb <= 32) { buf |= (unsigned long long)take() << (32 - nb); nb += 32; }
    }
};

// The rare codeword paths of lc_dec_v3_kernel (codes longer than the LUT, the
// payload end, invalid codewords), kept out of line so the hot loop stays small.
// Returns sym | l << 32 | status << 40 (l = 0: no codeword; the reader is
// passed by value so the caller's stays in registers).
#define LC_V3_LONG_SMEM 2048          // symbols of codes longer than the LUT kept in shared memory
__device__ __noinline__ unsigned long long lc_v3_slow_symbol(const LcDecV3Tables &Ts, const LcDecTables *Tg,
                                                            const uint32_t *__restrict__ sorted,
                                                            const uint32_t *s_long, unsigned long0, unsigned nlong,
                                                            const LcBitReader<LcGlobSrc> br, unsigned bits_rel)
{
    int l = lc_long_len_fast(Ts, br.buf);
    if (l && l <= 32 && br.pos + (unsigned)l <= bits_rel) {
        const unsigned long long v = (br.buf >> 32) >> (32 - l);
        const unsigned long long idx = Ts.offset[l] + (v - Ts.first_code[l]);
        const uint32_t sym = idx - long0 < nlong ? s_long[idx - long0] : __ldg(sorted + idx);
        return sym | ((unsigned long long)l << 32);
    }
    int term = 0;
    uint32_t sym = 0;
    l = lc_next_symbol(*Tg, sorted, br, bits_rel, &sym, &term);
    if (!l) return (unsigned long long)(term == 4 ? 2 : term) << 40;
    return sym | ((unsigned long long)l << 32);
}

__global__ void __launch_bounds__(LC_V3_TPB) lc_dec_v3_kernel(LcDecParams P, const unsigned long long *__restrict__ sync,
                                                             const double *__restrict__ starts,
                                                             const unsigned long long *__restrict__ sesc,
                                                             unsigned long long nsync, unsigned long long m,
                                                             double first_value, double delta,
                                                             const double *__restrict__ esc_val,
                                                             const unsigned long long *__restrict__ esc_idx,
                                                             unsigned long long n_esc, double *__restrict__ out,
                                                             LcV3Final *fin)
{
    __shared__ LcDecV3Tables Ts;
    __shared__ uint32_t s_long[LC_V3_LONG_SMEM];         // canonical symbols of the long codes
    __shared__ uint32_t s_ring[LC_V3_TPB * 8];           // fast path: per-lane prefetch ring (2 groups)
    extern __shared__ double v3_stage[];                 // [warps][32 rows][33]
    const LcDecTables *Tg = P.T;
    // long codes (> LC_LUT_BITS) are the tail of the canonical symbol order
    const int tml = Tg->max_len;
    const unsigned long0 = tml > LC_LUT_BITS ? (unsigned)Tg->offset[LC_LUT_BITS + 1] : 0u;
    const unsigned nlong_all = tml > LC_LUT_BITS ? (unsigned)Tg->used - long0 : 0u;
    // blocks with codes of 13..32 bits: s_long holds the symbols of the 13..16-bit codes by
    // 16-bit prefix instead (sym16, beside Ts.len16), so the straight-line walk resolves them
    // with two independent loads; longer codes then read `sorted` from global memory
    const bool cand16 = tml > LC_LUT_BITS && tml <= 32;
    const unsigned nlong = cand16 ? 0u : (nlong_all <= LC_V3_LONG_SMEM ? nlong_all : 0u);
    for (unsigned i = threadIdx.x; i < nlong; i += blockDim.x) s_long[i] = __ldg(P.sorted + long0 + i);
    if (threadIdx.x == 0) { Ts.max_len = Tg->max_len; Ts.canon = Tg->canon; Ts.s16 = Tg->s16; }
    for (int i = threadIdx.x; i < 34; i += blockDim.x) Ts.lim[i] = Tg->lim[i];
    for (int i = threadIdx.x; i < 66; i += blockDim.x) { Ts.first_code[i] = Tg->first_code[i]; Ts.offset[i] = Tg->offset[i]; }
    for (int i = threadIdx.x; i < (1 << LC_LUT_BITS) / 4; i += blockDim.x)
        reinterpret_cast<uint4 *>(Ts.lut)[i] = __ldg(reinterpret_cast<const uint4 *>(Tg->lut) + i);
    for (int i = threadIdx.x; i < LC_L16 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(Ts.len16)[i] = __ldg(reinterpret_cast<const uint4 *>(Tg->len16) + i);
    __syncthreads();
    uint16_t *sym16 = reinterpret_cast<uint16_t *>(s_long);
    bool m16 = cand16;
    if (cand16) {
        static_assert(LC_L16 * sizeof(uint16_t) <= LC_V3_LONG_SMEM * sizeof(uint32_t), "sym16 must fit s_long");
        int big = 0;
        for (int i = threadIdx.x; i < LC_L16; i += blockDim.x) {
            const int l = Ts.len16[i];
            uint32_t sy = 0;
            if (l) {
                const unsigned long long v = (unsigned long long)(Ts.s16 + (unsigned)i) >> (16 - l);
                sy = __ldg(P.sorted + Ts.offset[l] + (v - Ts.first_code[l]));
                big |= sy > 0xffffu;
            }
            sym16[i] = (uint16_t)sy;
        }
        m16 = __syncthreads_or(big) == 0;                // symbols beyond u16 (u32 codes): table unused
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double *stg = v3_stage + (size_t)wid * 32 * 33;
    double *myrow = stg + lane * 33;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[0] = first_value;
        if (nsync && lc_bits(starts[0]) != lc_bits(first_value)) atomicExch(&fin->status, 6);
    }
    const unsigned long long ngroups = (nsync + 31) / 32;
    // groups are dealt round-robin over the CTAs (group = warp slot * grid + CTA): with the grid
    // at one resident wave every SM gets the same number of groups +-1 (with 8 consecutive
    // groups per CTA, 2^26 elements put 16 warps on 108 SMs and 8 on the other 40)
    for (unsigned long long g = (unsigned long long)wid * gridDim.x + blockIdx.x; g < ngroups;
         g += (unsigned long long)gridDim.x * (LC_V3_TPB / 32)) {
        const unsigned long long j = g * 32 + lane;      // this lane's interval
        const bool live = j < nsync;
        const unsigned long long o0 = j * LC_SYNC_K;
        unsigned todo = live ? (unsigned)min((unsigned long long)LC_SYNC_K, m - o0) : 0u;
        const unsigned long long s0 = live ? sync[j] : 0ull;
        const unsigned long long s1 = live ? (j + 1 < nsync ? sync[j + 1] : P.bits) : 0ull;
        int bad = 0;
        if (live && (s0 > s1 || s1 > P.bits || (j == 0 && s0 != 0))) { bad = 6; todo = 0; }
        const unsigned long long wbase = s0 & ~127ull;    // 16-byte group of the start
        const unsigned bits_rel = lc_bits_rel(P.bits, wbase);
        LcV3Reader br;
        br.g4 = reinterpret_cast<const uint4 *>(P.payload + wbase / 32);
        br.pos = 0;
        if (todo) br.seek((unsigned)(s0 - wbase));
        double r = live ? starts[j] : 0.0;
        unsigned long long e = live ? sesc[j] : 0ull;
        int fl0 = 0, fl1 = 0;
        // Fast path: in a block whose codes are at most 32 bits long, a warp without a malformed
        // table entry runs a straight-line walk: no payload-end branches, codes longer than the
        // LUT and escapes resolved where they occur (rare branches); refills come from a per-lane shared-memory ring
        // kept two 16-byte groups ahead by asynchronous loads.  Invalid codewords, escape
        // codes or table disagreements are caught after the walk (status 1 / 6).
        {
            // the block's last interval (possibly short) and the lanes behind it take part too
            // (tail): otherwise the last warp alone would run the slower general walk and set the
            // kernel's duration (measured: 350 instead of 175 us at 2^26, eb 1e-3)
            const bool lastiv = live && j + 1 == nsync;
            const bool full = !live || (!bad && (lastiv || todo == LC_SYNC_K));
            const bool tail = __any_sync(0xffffffffu, !live || lastiv);
            if (Ts.max_len <= 32 && __all_sync(0xffffffffu, full)) {
                const unsigned f = (unsigned)(lane >> 2) & 7u;             // ring swizzle (bank spread)
                uint32_t *ring = s_ring + threadIdx.x * 8;
                const uint4 *g4 = reinterpret_cast<const uint4 *>(P.payload + wbase / 32);
                const unsigned p0 = (unsigned)(s0 - wbase);
                unsigned next = p0 >> 5;                                   // next word to buffer
                {
                    const unsigned gi = next >> 2;
                    const uint4 a = __ldg(g4 + gi), b = __ldg(g4 + gi + 1);
                    const unsigned sa = (gi & 1u) * 4u, sbb = ((gi + 1u) & 1u) * 4u;
                    ring[(sa + 0) ^ f] = a.x; ring[(sa + 1) ^ f] = a.y; ring[(sa + 2) ^ f] = a.z; ring[(sa + 3) ^ f] = a.w;
                    ring[(sbb + 0) ^ f] = b.x; ring[(sbb + 1) ^ f] = b.y; ring[(sbb + 2) ^ f] = b.z; ring[(sbb + 3) ^ f] = b.w;
                }
                uint4 pend = __ldg(g4 + (next >> 2) + 2);
                __syncwarp();
                auto word = [&](unsigned i) { return __byte_perm(ring[(i & 7u) ^ f], 0, 0x0123); };
                const int sh = (int)(p0 & 31);
                unsigned long long buf = (((unsigned long long)word(next) << 32) | word(next + 1)) << sh;
                int nb = 64 - sh;
                next += 2;
                unsigned pos = p0;
                bool inv = false;
                auto turn = [&]() {                                        // entering group next >> 2
                    const unsigned gg = next >> 2, sl = ((gg + 1u) & 1u) * 4u;
                    ring[(sl + 0) ^ f] = pend.x; ring[(sl + 1) ^ f] = pend.y;
                    ring[(sl + 2) ^ f] = pend.z; ring[(sl + 3) ^ f] = pend.w;
                    pend = __ldg(g4 + gg + 2);
                };
                if ((next & 3u) < 2u) turn();                              // both start words were consumed
                if (nb <= 32) {
                    buf |= (unsigned long long)word(next) << (32 - nb);
                    nb += 32;
                    ++next;
                    if ((next & 3u) == 0) turn();
                }
                double *orow = out + j * LC_SYNC_K + 1 - lane * LC_SYNC_K;   // + rr * 1024 + lane below
                // The walk is bound by the latency of one warp's dependent steps, where every branch in
                // the loop costs a pipeline bubble even when it is never taken: the escape and
                // long-code branches are compiled in only for warps / blocks that can need them.
                auto walk = [&](auto esc_tag, auto long_tag) {
                constexpr bool ESC = decltype(esc_tag)::value, LONG = decltype(long_tag)::value;
                uint32_t wnext = word(next);                               // the ring word the next refill takes
                for (unsigned sb = 0; sb < LC_SYNC_K; sb += 32) {
#pragma unroll 4
                    for (unsigned t = 0; t < 32; ++t) {
                        const bool act = !tail || sb + t < todo;           // tail: the walk stops at the interval's end
                        const uint32_t e1 = Ts.lut[(unsigned)(buf >> (64 - LC_LUT_BITS))];
                        uint32_t sym = act ? e1 & 0xffffffu : 1u;          // 1: m = 0
                        int l = (int)(e1 >> 24);
                        if (LONG && act && l > LC_LUT_BITS) {              // a code longer than the LUT (<= 32 bits here)
                            const unsigned i16 = (unsigned)(buf >> 48) - Ts.s16;
                            const int l16 = (m16 && i16 < (unsigned)LC_L16) ? (int)Ts.len16[i16] : 0;
                            const int l2 = l16 ? l16 : lc_long_len_fast(Ts, buf);   // 13..16 bits by table, longer by the limits
                            if (l16) {
                                sym = sym16[i16];
                                l = l16;
                            } else if (l2 > 0 && l2 <= 32) {
                                const unsigned long long v = (buf >> 32) >> (32 - l2);
                                const unsigned long long idx = Ts.offset[l2] + (v - Ts.first_code[l2]);
                                sym = idx - long0 < nlong ? s_long[idx - long0] : __ldg(P.sorted + idx);
                                l = l2;
                            } else {
                            LcBitReader<LcGlobSrc> gr;
                            gr.src.w = P.payload + wbase / 32;
                            gr.buf = buf; gr.nb = nb; gr.pos = pos; gr.next = next;
                            const unsigned long long sl =
                                lc_v3_slow_symbol(Ts, Tg, P.sorted, s_long, long0, nlong, gr, bits_rel);
                            sym = (uint32_t)sl;
                            l = (int)((sl >> 32) & 0xff);
                            if (l == 0 || l > 32) { inv = true; l = 1; sym = 1u; }   // no codeword here: flagged, walk on
                            }
                        }
                        const int lc = act ? (LONG ? l : (l & 15)) : 0;
                        buf <<= lc;
                        nb -= lc;
                        pos += lc;
                        // refill without a branch: the next ring word is always at hand (loaded one step
                        // ahead, so its shared-memory latency is off the dependent walk); only the ring
                        // turn every fourth refill branches
                        const bool rf = nb <= 32;
                        buf |= rf ? (unsigned long long)wnext << ((32 - nb) & 63) : 0ull;
                        nb += rf ? 32 : 0;
                        next += rf ? 1u : 0u;
                        if (rf && (next & 3u) == 0) turn();
                        wnext = word(next);
                        if (ESC && act && sym == 0u) {                     // escape (compressor.py:365-369): rare
                            const unsigned long long posn = o0 + sb + t + 1;   // element index
                            if (e < n_esc) {
                                r = __ldg(esc_val + e);
                                fl1 |= __ldg(esc_idx + e) != posn;
                            } else {
                                fl0 = 1;
                            }
                            ++e;
                        }
                        if (!ESC) e += (act && sym == 0u) ? 1ull : 0ull;  // an escape the table does not know: the end check fails
                        if (!LONG) inv |= act && l > LC_LUT_BITS;
                        const uint32_t zz = sym - 1u;                      // compressor.py:370-374
                        const int mm = (int)(zz >> 1) ^ -(int)(zz & 1u);
                        const double inc = LC_MUL((double)mm, delta);
                        if (sym > 1u) r = LC_ADD(r, inc);
                        myrow[t] = r;
                    }
                    __syncwarp();
                    if (!tail) {
#pragma unroll 4
                        for (int rr = 0; rr < 32; ++rr)
                            __stcs(orow + (size_t)rr * LC_SYNC_K + sb + lane, stg[rr * 33 + lane]);
                    } else {
                        for (int rr = 0; rr < 32; ++rr) {
                            const unsigned long long jr = g * 32 + rr;
                            if (jr >= nsync) break;
                            const unsigned long long lim = min((unsigned long long)LC_SYNC_K, m - jr * LC_SYNC_K);
                            if (sb + lane < lim) __stcs(out + jr * LC_SYNC_K + sb + 1 + lane, stg[rr * 33 + lane]);
                        }
                    }
                    __syncwarp();
                }
                };
                const bool has_esc = __any_sync(0xffffffffu, live && (lastiv ? e != n_esc : sesc[j + 1] != e));
                const bool has_long = Ts.max_len > LC_LUT_BITS;
                if (has_esc) {
                    if (has_long) walk(std::true_type{}, std::true_type{});
                    else walk(std::true_type{}, std::false_type{});
                } else {
                    if (has_long) walk(std::false_type{}, std::true_type{});
                    else walk(std::false_type{}, std::false_type{});
                }
                if (live) {
                    if (inv) atomicExch(&fin->status, 1);
                    else if (wbase + pos != s1 || (!lastiv && (lc_bits(r) != lc_bits(starts[j + 1]) || e != sesc[j + 1])))
                        atomicExch(&fin->status, 6);
                    if (fl0) atomicExch(&fin->esc_flags[0], 1);
                    if (fl1) atomicExch(&fin->esc_flags[1], 1);
                    if (lastiv) fin->esc_total = (long long)e;
                }
                continue;
            }
        }
        const unsigned wsteps = __reduce_max_sync(0xffffffffu, todo);
        for (unsigned sb = 0; sb < wsteps; sb += 32) {
            const unsigned nt = todo > sb ? min(32u, todo - sb) : 0u;   // symbols of this block
            // Lanes step in lockstep (32 steps, predicated by `act`).  The common step is a
            // short straight line (LUT lookup, 64-bit shift, one reference add); the rare
            // paths -- long codes / payload end, escapes, buffer refills and prefetch-ring
            // turns -- are warp-uniform branches entered only when some lane needs them.
#pragma unroll 1
            for (unsigned t = 0; t < 32; ++t) {
                const bool act = t < nt && !bad;
                const uint32_t e1 = Ts.lut[(unsigned)(br.buf >> (64 - LC_LUT_BITS))];
                uint32_t sym = e1 & 0xffffffu;
                int l = (int)(e1 >> 24);
                const bool slow = act && (l > LC_LUT_BITS || br.pos + (unsigned)l > bits_rel);
                if (__any_sync(0xffffffffu, slow)) {
                    if (slow) {
                        LcBitReader<LcGlobSrc> gr;                    // the same position, global reads
                        gr.src.w = P.payload + wbase / 32;
                        gr.buf = br.buf; gr.nb = br.nb; gr.pos = br.pos; gr.next = br.next;
                        const unsigned long long sl =
                            lc_v3_slow_symbol(Ts, Tg, P.sorted, s_long, long0, nlong, gr, bits_rel);
                        sym = (uint32_t)sl;
                        l = (int)((sl >> 32) & 0xff);
                        if (!l) { bad = (int)(sl >> 40); todo = 0; }
                        else if (l >= br.nb) { br.seek(br.pos + l); l = 0; }   // consumed by the seek
                    }
                }
                const bool go = act && !bad;
                const int lc = go ? l : 0;
                br.buf <<= lc;
                br.nb -= lc;
                br.pos += lc;
                const bool rf = br.nb <= 32;
                if (__any_sync(0xffffffffu, rf)) {
                    if (rf) {
                        br.buf |= (unsigned long long)LcV3Reader::pick(br.cur, br.next & 3u) << (32 - br.nb);
                        br.nb += 32;
                        ++br.next;
                    }
                    const bool turn = rf && (br.next & 3u) == 0;      // the current group is used up
                    if (__any_sync(0xffffffffu, turn)) {
                        if (turn) {
                            br.cur = br.n1;
                            br.n1 = br.n2;
                            br.n2 = __ldg(br.g4 + (br.next >> 2) + 2);
                        }
                    }
                }
                const bool esc = go && sym == 0;
                if (__any_sync(0xffffffffu, esc)) {
                    if (esc) {                                        // compressor.py:365-369
                        const unsigned long long pos = o0 + sb + t + 1;   // element index
                        if (e < n_esc) {
                            r = esc_val[e];
                            fl1 |= esc_idx[e] != pos;
                        } else {
                            fl0 = 1;
                        }
                        ++e;
                    }
                }
                const uint32_t zz = sym - 1u;                          // :370-374 (m != 0 iff sym > 1)
                const int mm = (int)(zz >> 1) ^ -(int)(zz & 1u);
                const double inc = LC_MUL((double)mm, delta);
                if (go && sym > 1u) r = LC_ADD(r, inc);
                myrow[t] = r;
            }
            if (bad) todo = 0;
            __syncwarp();
            // rows: lane L's values go to out[o0(L) + sb + 1 ...]
            for (int rr = 0; rr < 32; ++rr) {
                const unsigned long long jr = g * 32 + rr;
                if (jr >= nsync) break;
                const unsigned long long base = jr * LC_SYNC_K + sb + 1;
                const unsigned long long lim = min((unsigned long long)LC_SYNC_K, m - jr * LC_SYNC_K);
                if (sb + lane < lim) __stcs(out + base + lane, stg[rr * 33 + lane]);
            }
            __syncwarp();
        }
        if (live) {
            if (bad) atomicExch(&fin->status, bad);
            else if (wbase + br.pos != s1) atomicExch(&fin->status, 6);
            else if (j + 1 < nsync && (lc_bits(r) != lc_bits(starts[j + 1]) || e != sesc[j + 1]))
                atomicExch(&fin->status, 6);
            if (fl0) atomicExch(&fin->esc_flags[0], 1);
            if (fl1) atomicExch(&fin->esc_flags[1], 1);
            if (j + 1 == nsync) fin->esc_total = (long long)e;
        }
    }
}

// Resolve the reference status (huffman.py:114-132) from the segment walk.
__global__ void lc_dec_status_kernel(const LcSeg *__restrict__ seg, const unsigned long long *__restrict__ off,
                                     const unsigned long long *__restrict__ total_and_term,
                                     const unsigned long long *__restrict__ end_pos, unsigned long long m,
                                     unsigned long long bits, int *__restrict__ status)
{
    const unsigned long long ft = total_and_term[1];
    unsigned long long K = total_and_term[0];   // symbols on the path when no anomaly
    int term = 4;
    if (ft != ~0ULL) { K = off[ft] + seg[ft].count; term = seg[ft].term; }
    int st;
    if (m <= K) st = (*end_pos == bits) ? 0 : 3;
    else st = (term == 4) ? 2 : term;           // ran out exactly at bit_length -> exhausted
    *status = st;
}

// ---------------------------------------------------------------------------
// reconstruction

struct LcSegScan {             // running state of the escape-segmented m-prefix
    long long sum;              // sum of m since the last escape (or the start)
    long long cnt;              // escape codes so far
    int has;                    // an escape occurred
    int moved;                  // a non-zero m occurred since the last escape
};

__device__ __forceinline__ LcSegScan lc_segscan_op(const LcSegScan &a, const LcSegScan &b)
{
    LcSegScan r;
    r.sum = b.has ? b.sum : a.sum + b.sum;
    r.cnt = a.cnt + b.cnt;
    r.has = a.has | b.has;
    r.moved = b.has ? b.moved : (a.moved | b.moved);
    return r;
}

// look-back descriptor of one reconstruction tile: status 1 = aggregate, 2 = inclusive
struct LcSegDesc {
    int st;
    int pad;
    LcSegScan agg, incl;
};

__device__ __forceinline__ LcSegScan lc_shfl_down_seg(const LcSegScan &v, int o)
{
    LcSegScan r;
    r.sum = __shfl_down_sync(0xffffffffu, v.sum, o);
    r.cnt = __shfl_down_sync(0xffffffffu, v.cnt, o);
    r.has = __shfl_down_sync(0xffffffffu, v.has, o);
    r.moved = __shfl_down_sync(0xffffffffu, v.moved, o);
    return r;
}


struct LcRecParams {
    const void *codes;
    int code_bytes;
    uint64_t n;                 // elements (codes: n-1)
    double delta;
    double first_value;
    const double *esc_val;
    const unsigned long long *esc_idx;
    unsigned long long n_esc;
    int64_t first_chunk;
    double anchor_val;          // exact value at position first_chunk*L
    long long anchor_cnt;       // escapes before position first_chunk*L (inclusive)
    int64_t nchunks, ntiles;
    double *out;
    unsigned long long *first_bad;
    double *bad_end;
    long long *chunk_esc;       // escapes up to each chunk's start (inclusive of position cL)
    int *esc_flags;             // [0] more escape codes than values, [1] position mismatch
    const int *abort_a, *abort_b;   // decode status / cascade flag: non-zero -> kernels exit (no host sync before)
    long long inject_chunk;     // test hook: perturb this chunk's predicted start (fresh launch only), -1 off
};

__device__ __forceinline__ bool lc_rec_aborted(const LcRecParams &P)
{
    return (P.abort_a && *(volatile const int *)P.abort_a) || (P.abort_b && *(volatile const int *)P.abort_b);
}

__device__ __forceinline__ int lc_code_m(uint32_t code) { return lc_unzigzag(code); }
// the same for a non-escape code (code 0 gives garbage; callers replace that step's value)
__device__ __forceinline__ int lc_code_m_nz(uint32_t code)
{
    const uint32_t zz = code - 1u;
    return (int)(zz >> 1) ^ -(int)(zz & 1u);
}

// ---------------------------------------------------------------------------
// Split reconstruction: RA (segmented m-prefix by block scan + look-back, guess
// chains + maps), map scan (lc_map_scan_kernel), RB exact chain.


struct LcRecSplit {
    LcSegScan *tile_seg;      // [ntiles] RA: tile aggregate of the segmented m-prefix
    LcSegScan *tile_in;       // [ntiles] RA: state at each tile start
    LcSegDesc *seg_desc;      // [ntiles] RA look-back descriptors (status zeroed per launch)
    unsigned long long *tile_ctr;   // RA dynamic tile counter (zeroed per launch)
    OffMap *tile_agg;         // [ntiles] RA output
    double *tile_D;           // [ntiles + 1] map scan output
    LcChunkPred pred;         // RA -> RB
};

// This thread's chunk codes (32 consecutive) with 16-byte loads; the tail
// chunk falls back to scalar loads.  v[j] = code j (0 past the end).
__device__ __forceinline__ void lc_load_chunk_codes(const LcRecParams &P, long long p0, int len, uint32_t (&v)[LC_L])
{
    if (len == LC_L) {
        if (P.code_bytes == 2) {
            const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint16_t *>(P.codes) + p0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint4 q = __ldg(src + k);
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    v[8 * k + 2 * h] = w4[h] & 0xffffu;
                    v[8 * k + 2 * h + 1] = w4[h] >> 16;
                }
            }
        } else {
            const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(P.codes) + p0);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint4 q = __ldg(src + k);
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < LC_L; ++j) {
            uint32_t c = 0;
            if (j < len) c = P.code_bytes == 2 ? (uint32_t)reinterpret_cast<const uint16_t *>(P.codes)[p0 + j]
                                               : reinterpret_cast<const uint32_t *>(P.codes)[p0 + j];
            v[j] = c;
        }
    }
}

// Codes of the tile into padded smem rows (row = this thread's chunk).
__device__ __forceinline__ void lc_load_codes_tile(const LcRecParams &P, long long pbeg, uint32_t *cs)
{
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    const long long p0 = pbeg + (long long)tid * LC_L;
    const int len = (int)max(0LL, min((long long)LC_L, nel - p0));
    uint32_t v[LC_L];
    lc_load_chunk_codes(P, p0, len, v);
    uint32_t *row = cs + tid * LC_ROW;
#pragma unroll
    for (int j = 0; j < LC_L; ++j) row[j] = v[j];
}

// L2 prefetch of tile t's codes (rec kernels run tiles t, t + gridDim.x, ...)
__device__ __forceinline__ void lc_prefetch_codes_tile(const LcRecParams &P, long long t)
{
    if (t >= P.ntiles) return;
    const long long p0 = (P.first_chunk + t * LC_TPB) * LC_L;
    const long long nel = (long long)P.n - 1;
    const long long cnt = min((long long)LC_TILE, nel - p0);
    if (cnt > 0) lc_prefetch_bytes(reinterpret_cast<const char *>(P.codes) + p0 * P.code_bytes, cnt * P.code_bytes);
}

__device__ __forceinline__ LcSegScan lc_shfl_up_seg(const LcSegScan &v, int o)
{
    LcSegScan r;
    r.sum = __shfl_up_sync(0xffffffffu, v.sum, o);
    r.cnt = __shfl_up_sync(0xffffffffu, v.cnt, o);
    r.has = __shfl_up_sync(0xffffffffu, v.has, o);
    r.moved = __shfl_up_sync(0xffffffffu, v.moved, o);
    return r;
}

// block-wide exclusive scan of chunk segscan states; returns exclusive, *agg = tile total
__device__ __forceinline__ LcSegScan lc_block_segscan(const LcSegScan &mine, LcSegScan *wseg, LcSegScan *agg)
{
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    LcSegScan inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const LcSegScan up = lc_shfl_up_seg(inc, o);
        if (lane >= o) inc = lc_segscan_op(up, inc);
    }
    if (lane == 31) wseg[wid] = inc;
    __syncthreads();
    if (tid == 0)
        for (int w = 1; w < LC_TPB / 32; ++w) wseg[w] = lc_segscan_op(wseg[w - 1], wseg[w]);
    __syncthreads();
    if (wid > 0) inc = lc_segscan_op(wseg[wid - 1], inc);
    LcSegScan exc = lc_shfl_up_seg(inc, 1);
    if (lane == 0) {
        if (wid > 0) exc = wseg[wid - 1];
        else { exc.sum = 0; exc.cnt = 0; exc.has = 0; exc.moved = 0; }
    }
    *agg = wseg[LC_TPB / 32 - 1];
    return exc;
}

// RA: tiles in claim order (dynamic counter, so every tile a CTA waits for
// was claimed earlier by a running CTA).  Each tile derives the escape-
// segmented m-prefix of its chunks from its codes (block scan) and the state at
// the tile start by a decoupled look-back over the tiles' aggregates; then
// guess chains, flags, compacted replays and the in-tile map scan.
__global__ void __launch_bounds__(LC_TPB, 4) lc_rec_a_kernel(LcRecParams P, LcRecSplit S)
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    uint32_t *cs = reinterpret_cast<uint32_t *>(lc_dyn_smem);
    __shared__ OffMap warp_agg[LC_TPB / 32];
    __shared__ LcReplayItem s_rq[LC_TPB];
    __shared__ int s_rcnt[LC_TPB / 32];
    __shared__ LcSegScan wseg[LC_TPB / 32];
    __shared__ LcSegScan s_tin;
    __shared__ long long s_tile;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long nel = (long long)P.n - 1;
    if (lc_rec_aborted(P)) return;
    for (;;) {
        __syncthreads();                                 // the previous tile is done with smem
        if (tid == 0) s_tile = (long long)atomicAdd(S.tile_ctr, 1ull);
        __syncthreads();
        const long long t = s_tile;
        if (t >= P.ntiles) break;
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long c = cbeg + tid;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - c * LC_L) : 0;
        LcSegScan mine; mine.sum = 0; mine.cnt = 0; mine.has = 0; mine.moved = 0;
        {
            uint32_t v[LC_L];
            lc_load_chunk_codes(P, c * LC_L, len, v);
            uint32_t *row = cs + tid * LC_ROW;
#pragma unroll
            for (int j = 0; j < LC_L; ++j) {
                row[j] = v[j];
                if (j < len) {
                    const uint32_t code = v[j];
                    if (code == 0) { mine.sum = 0; mine.cnt += 1; mine.has = 1; mine.moved = 0; }
                    else { const int mm = lc_code_m(code); mine.sum += mm; mine.moved |= (mm != 0); }
                }
            }
        }
        lc_prefetch_codes_tile(P, t + 1);
        LcSegScan agg;
        const LcSegScan exc = lc_block_segscan(mine, wseg, &agg);      // barriers inside
        if (wid == 0) {
            LcSegDesc *d = S.seg_desc + t;
            if (lane == 0) {
                d->agg = agg;
                __threadfence();
                st_release(&d->st, 1);
            }
            LcSegScan ident; ident.sum = 0; ident.cnt = 0; ident.has = 0; ident.moved = 0;
            LcSegScan first; first.sum = 0; first.cnt = P.anchor_cnt; first.has = 1; first.moved = 0;   // launch anchor
            const LcSegScan pre = lc_lookback_warp<LcSegScan>(
                t, ident, [](const LcSegScan &x, const LcSegScan &y) { return lc_segscan_op(x, y); },
                [](const LcSegScan &v, int o) { return lc_shfl_down_seg(v, o); },
                [&](long long k) { return ld_acquire(&S.seg_desc[k].st); },
                [&](long long k, int st) {
                    const LcSegDesc *q = S.seg_desc + k;
                    LcSegScan r;
                    const LcSegScan *src = st == 2 ? &q->incl : &q->agg;
                    r.sum = __ldcg(&src->sum); r.cnt = __ldcg(&src->cnt);
                    r.has = __ldcg(&src->has); r.moved = __ldcg(&src->moved);
                    return r;
                }, &first);
            if (lane == 0) {
                d->incl = lc_segscan_op(pre, agg);
                __threadfence();
                st_release(&d->st, 2);
                s_tin = pre;
                S.tile_in[t] = pre;
                S.tile_seg[t] = agg;
            }
        }
        __syncthreads();
        const uint32_t *crow = cs + tid * LC_ROW;
        const LcSegScan tin = s_tin;
        LcSegScan before = tin, after = tin;
        if (len > 0) {
            before = lc_segscan_op(tin, exc);
            if (c + 1 < P.nchunks) after = lc_segscan_op(before, mine);
        }
        auto anchor_of = [&](const LcSegScan &s) -> double {
            if (s.cnt > P.anchor_cnt) {
                const long long e = s.cnt - 1;
                return e < (long long)P.n_esc ? P.esc_val[e] : 0.0;
            }
            return P.anchor_val;
        };
        auto guess_of = [&](const LcSegScan &s) -> double {
            const double a = anchor_of(s);
            if (!s.moved) return a;
            const double g = LC_ADD(a, LC_MUL((double)s.sum, P.delta));
            return isfinite(g) ? g : a;
        };
        const double g0 = guess_of(before);
        const double g1 = guess_of(after);
        // guess chain with superset event flags; flagged chunks are replayed below
        // by a compacted queue of threads
        OffMap H;
        bool need = false;
        unsigned mask = 0u;
        double r = g0, rs = g0;                      // rs: chain value before the first flagged step
        if (len > 0) {
            P.chunk_esc[c] = before.cnt;
            long long e = before.cnt;
            LcFlags F;
            lc_flags_init(F, g0);
            int anyesc = 0;
            for (int j = 0; j < len; ++j) {
                const uint32_t code = crow[j];
                const int m = lc_code_m_nz(code);            // escapes (code 0) are replaced below
                const double inc_ = LC_MUL((double)m, P.delta);
                double rn = m != 0 ? LC_ADD(r, inc_) : r;
                if (code == 0) { rn = e < (long long)P.n_esc ? P.esc_val[e] : 0.0; ++e; anyesc = 1; }
                const bool f = lc_flag_test(F, r, inc_, rn);
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
            uint32_t *rw = cs + lc_replay_ch(it) * LC_ROW;
            const int j0 = __ffs(it.mask) - 1, j1 = 31 - __clz(it.mask);
            OffMap Hr = lc_map_identity(lc_replay_ulp(it));
            double r2 = it.rs;
            for (int j = j0; j <= j1; ++j) {
                const int m = lc_code_m(rw[j]);              // no escapes in replayed chunks
                if (m != 0) {
                    const double inc_ = LC_MUL((double)m, P.delta);
                    const double rn = LC_ADD(r2, inc_);
                    if ((it.mask >> j) & 1u) lc_map_step(Hr, r2, inc_, rn);
                    r2 = rn;
                }
            }
            lc_map_to_words(rw, Hr);
        });
        if (need) H = lc_map_from_words(crow);
        if (len > 0 && c + 1 < P.nchunks) lc_map_shift_out(H, LC_SUB(r, g1));
        OffMap inc_map = H;
        lc_warp_scan_maps(inc_map);
        if (lane == 31) warp_agg[wid] = inc_map;
        __syncthreads();
        lc_scan_warp_maps(warp_agg, LC_TPB / 32);
        __syncthreads();
        // shuffle first (the warp is converged after the scan), compose per lane afterwards:
        // no shuffle may follow a per-lane composition (see lc_warp_scan_maps)
        OffMap exc_map = lc_shfl_up_map(inc_map, 1);
        if (lane == 0) exc_map = lc_map_neutral();
        if (wid > 0) exc_map = lc_map_compose(exc_map, warp_agg[wid - 1]);
        if (len > 0) {
            S.pred.kind[c] = exc_map.kind;
            S.pred.B[c] = exc_map.B;
            S.pred.t0[c] = exc_map.t0;
            S.pred.t1[c] = exc_map.t1;
            S.pred.y[c] = exc_map.y;
            S.pred.g0[c] = g0;
        }
        if (tid == 0) S.tile_agg[t] = warp_agg[LC_TPB / 32 - 1];
    }
}

// Exact chain (compressor.py:360-375): codes straight into registers (no smem
// staging), all per-chunk loads issued together, results transposed through
// padded smem rows and written with 16-byte streaming stores.
template <int CB>
__global__ void __launch_bounds__(LC_TPB, 3) lc_rec_b_kernel(LcRecParams P, LcRecSplit S)
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    double *ys = reinterpret_cast<double *>(lc_dyn_smem);
    __shared__ double starts[LC_TPB + 1];
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    if (lc_rec_aborted(P)) return;
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long pbeg = cbeg * LC_L;
        const long long c = cbeg + tid;
        const long long p0 = c * LC_L;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - p0) : 0;
        uint32_t v[LC_L];
        if (len == LC_L) {
            if (CB == 2) {
                const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint16_t *>(P.codes) + p0);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint4 q = __ldcs(src + k);
                    const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) { v[8 * k + 2 * h] = w4[h] & 0xffffu; v[8 * k + 2 * h + 1] = w4[h] >> 16; }
                }
            } else {
                const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(P.codes) + p0);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint4 q = __ldcs(src + k);
                    v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < LC_L; ++j)
                v[j] = j < len ? (CB == 2 ? (uint32_t)reinterpret_cast<const uint16_t *>(P.codes)[p0 + j]
                                          : reinterpret_cast<const uint32_t *>(P.codes)[p0 + j]) : 1u;
        }
        if (t + gridDim.x < P.ntiles) {                      // next tile's inputs
            const long long cn = P.first_chunk + (t + gridDim.x) * LC_TPB;
            lc_prefetch_codes_tile(P, t + gridDim.x);
            lc_prefetch_bytes(S.pred.kind + cn, LC_TPB * sizeof(int));
            lc_prefetch_bytes(S.pred.B + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(S.pred.t0 + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(S.pred.t1 + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(S.pred.y + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(S.pred.g0 + cn, LC_TPB * sizeof(double));
            lc_prefetch_bytes(P.chunk_esc + cn, LC_TPB * sizeof(long long));
        }
        double start = 0.0;
        long long e = 0;
        if (len > 0) {
            OffMap m;
            m.kind = S.pred.kind[c]; m.B = S.pred.B[c]; m.t0 = S.pred.t0[c]; m.t1 = S.pred.t1[c]; m.y = S.pred.y[c];
            m.v = 0.0; m.og = 0.0;
            const double g0 = S.pred.g0[c];
            e = P.chunk_esc[c];
            start = lc_apply_offset(g0, lc_map_eval(m, S.tile_D[t]));
            // test hook (lc_ctx_set_option LC_OPT_INJECT_REC): a wrong prediction for this
            // chunk, so its predecessor's end check fails and the host relaunches
            if (c == P.inject_chunk && P.first_chunk == 0) start = lc_from_bits(lc_bits(start) ^ 1);
        }
        __syncthreads();                                 // previous tile's ys/starts reads are done
        starts[tid] = start;
        if (tid == LC_TPB - 1) {
            const long long cn = cbeg + LC_TPB;
            starts[LC_TPB] = (cn < P.nchunks) ? lc_apply_offset(S.pred.g0[cn], S.tile_D[t + 1]) : 0.0;
        }
        __syncthreads();
        double *yrow = ys + tid * LC_ROW;
        if (len > 0) {
            double r = start;
            auto step = [&](int j) {
                const uint32_t code = v[j];
                const int mm = lc_code_m_nz(code);                                   // code 0: replaced below
                double rn = mm != 0 ? LC_ADD(r, LC_MUL((double)mm, P.delta)) : r;   // compressor.py:371-374
                if (code == 0) {                                                     // :365-369
                    if (e < (long long)P.n_esc) {
                        rn = P.esc_val[e];
                        if (P.esc_idx[e] != (unsigned long long)(p0 + j + 1)) atomicExch(&P.esc_flags[1], 1);
                    } else {
                        atomicExch(&P.esc_flags[0], 1);
                    }
                    ++e;
                }
                yrow[j] = rn;
                r = rn;
            };
            if (len == LC_L) {                               // full chunk: no per-step length test
#pragma unroll
                for (int j = 0; j < LC_L; ++j) step(j);
            } else {
#pragma unroll
                for (int j = 0; j < LC_L; ++j) {
                    step(j);
                    if (j + 1 == len) break;
                }
            }
            if (c + 1 < P.nchunks && lc_bits(r) != lc_bits(starts[tid + 1])) {
                P.bad_end[c] = r;
                atomicMin(P.first_bad, (unsigned long long)(c + 1));
            }
        }
        __syncthreads();
        // out[pbeg + 1 + off], off = 0..8191: pairs (off, off+1) from smem, 16-byte
        // stores at even out positions (out + pbeg + 1 is 16-byte aligned iff out is
        // 8 mod 16, so the pairing phase follows the base address).
        const long long q0 = pbeg + 1;
        const int ph = (int)(((reinterpret_cast<uintptr_t>(P.out + q0)) >> 3) & 1);   // 1: first element alone
        const long long tile_n = min((long long)LC_TILE, nel - pbeg);
        if (ph && tid == 0) __stcs(P.out + q0, ys[0]);
#pragma unroll 4
        for (int k = 0; k < LC_L / 2; ++k) {
            const int off = ph + 2 * (k * LC_TPB + tid);
            if (off + 1 < tile_n) {
                const double a = ys[(off >> 5) * LC_ROW + (off & 31)];
                const double b = ys[((off + 1) >> 5) * LC_ROW + ((off + 1) & 31)];
                __stcs(reinterpret_cast<double2 *>(P.out + q0 + off), make_double2(a, b));
            } else if (off < tile_n) {
                __stcs(P.out + q0 + off, ys[(off >> 5) * LC_ROW + (off & 31)]);
            }
        }
    }
}

size_t lc_rec_a_smem_bytes() { return sizeof(uint32_t) * LC_TPB * LC_ROW; }
static size_t lc_dec_v3_smem() { return sizeof(double) * (LC_V3_TPB / 32) * 32 * 33; }
size_t lc_rec_b_smem_bytes() { return sizeof(double) * LC_TPB * LC_ROW; }


__global__ void lc_set_first_kernel(double *out, double v) { out[0] = v; }

// ---------------------------------------------------------------------------
// driver

struct LcBuf { void *p = nullptr; size_t cap = 0; };   // same as lc_api.cu
cudaError_t lc_reserve(LcBuf &b, size_t bytes);
int lc_fail(lc_ctx *ctx, cudaError_t e, const char *what, const char *file, int line);
cudaStream_t lc_stream(lc_ctx *ctx);
int lc_sm_count(lc_ctx *ctx);
void *lc_pinned(lc_ctx *ctx);
void lc_set_err(lc_ctx *ctx, const char *msg);
LcBuf *lc_dec_bufs(lc_ctx *ctx);
cudaEvent_t lc_ev(lc_ctx *ctx, int which);
cudaEvent_t lc_phase_ev(lc_ctx *ctx, int i);
void lc_count_launch(lc_ctx *ctx, int k);
void lc_set_kind(lc_ctx *ctx, int k);
int lc_debug_check(lc_ctx *ctx, const char *what, const char *file, int line);
long long lc_opt(lc_ctx *ctx, int key);
int *lc_dec_state(lc_ctx *ctx);

static int lc_reconstruct(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const double *esc_val_in,
                          uint64_t n_esc, double *out, int out_on_device, int64_t *esc_used, void *codes,
                          int code_bytes, const int *abort_a, const int *abort_b, int *abort_hit);
#define LC_RC_CASCADE (-100)   // lc_reconstruct: the decode needs general sync passes, redo

int lc_decompress_impl2(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value,
                        const uint8_t *code_lengths, uint64_t n_lengths, const uint8_t *payload,
                        uint64_t payload_bytes, uint64_t payload_bits, const uint64_t *esc_idx,
                        const double *esc_val, uint64_t n_esc, int inputs_on_device, double *out,
                        int out_on_device, int64_t *esc_used, const uint64_t *sync, uint64_t n_sync,
                        const double *sync_starts, const uint64_t *sync_esc)
{
    if (n < 2 || n_lengths == 0 || n_lengths > (1ull << 31) + 2 || payload_bits > 8 * payload_bytes) return 12;
    cudaStream_t st = lc_stream(ctx);
    LcBuf *B = lc_dec_bufs(ctx);      // ctx->dec[10]
    LcBuf &bpay = B[0], &blen = B[1], &beidx = B[2], &beval = B[3], &bout = B[4], &bcodes = B[5], &btab = B[6],
          &bsync = B[7], &baux = B[8], &baux2 = B[9];
    LC_CUDA_OK(cudaEventRecord(lc_ev(ctx, 0), st));
    const uint64_t m = n - 1;
    const uint64_t words = (payload_bytes + 3) / 4 + 4;
    // padded to whole sync-CTA ranges (bulk copies of up to 256 * 32 + 8 words)
    const uint64_t words_alloc = words + LC_DEC_TPB * 32 + LC_DEC_STAGE_PAD + 64;
    LC_CUDA_OK(lc_reserve(bpay, words_alloc * 4));
    // zero only the padding behind the payload (the copy writes the rest)
    LC_CUDA_OK(cudaMemsetAsync((char *)bpay.p + payload_bytes, 0, words_alloc * 4 - payload_bytes, st));
    LC_CUDA_OK(cudaMemcpyAsync(bpay.p, payload, payload_bytes,
                               inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    LC_CUDA_OK(lc_reserve(blen, n_lengths));
    LC_CUDA_OK(cudaMemcpyAsync(blen.p, code_lengths, n_lengths,
                               inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    LC_CUDA_OK(lc_reserve(beidx, (n_esc + 1) * 8));
    LC_CUDA_OK(lc_reserve(beval, (n_esc + 1) * 8));
    if (n_esc) {
        const cudaMemcpyKind k = inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        LC_CUDA_OK(cudaMemcpyAsync(beidx.p, esc_idx, n_esc * 8, k, st));
        LC_CUDA_OK(cudaMemcpyAsync(beval.p, esc_val, n_esc * 8, k, st));
    }
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 5), st));
    // tables
    LC_CUDA_OK(lc_reserve(btab, sizeof(LcDecTables) + n_lengths * 4 + 64));
    LcDecTables *T = (LcDecTables *)btab.p;
    uint32_t *sorted = (uint32_t *)((char *)btab.p + sizeof(LcDecTables));
    if (n_lengths <= LC_DEC_LEN_SMEM) {
        const size_t lsm = (n_lengths + 15) / 16 * 16;
        lc_dec_tables_kernel<true><<<1, 1024, lsm, st>>>((const uint8_t *)blen.p, (uint32_t)n_lengths, T, sorted);
    } else {
        lc_dec_tables_kernel<false><<<1, 1024, 0, st>>>((const uint8_t *)blen.p, (uint32_t)n_lengths, T, sorted);
    }
    { int _rc = lc_debug_check(ctx, "lc_dec_tables_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    lc_count_launch(ctx, 2);
    // Huffman decode
    const int code_bytes = n_lengths <= 65536 ? 2 : 4;
    LC_CUDA_OK(lc_reserve(bcodes, m * code_bytes + 16));
    if (sync && sync_starts && sync_esc) {              // v3: decode + reconstruct per sync interval
        LC_CUDA_OK(lc_reserve(baux, 256));
        LcV3Final *dfin = (LcV3Final *)((char *)baux.p + 64);
        LcV3Final *hfin = (LcV3Final *)((char *)lc_pinned(ctx) + 256);
        LC_CUDA_OK(lc_reserve(bsync, n_sync * 24 + 64));
        const cudaMemcpyKind k = inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        unsigned long long *dsync = (unsigned long long *)bsync.p;
        double *dstart = (double *)(dsync + n_sync);
        unsigned long long *desc = (unsigned long long *)(dstart + n_sync);
        LC_CUDA_OK(cudaMemcpyAsync(dsync, sync, n_sync * 8, k, st));
        LC_CUDA_OK(cudaMemcpyAsync(dstart, sync_starts, n_sync * 8, k, st));
        LC_CUDA_OK(cudaMemcpyAsync(desc, sync_esc, n_sync * 8, k, st));
        LC_CUDA_OK(cudaMemsetAsync(dfin, 0, sizeof(LcV3Final), st));
        double *dout = out;
        if (!out_on_device) {
            LC_CUDA_OK(lc_reserve(bout, n * 8));
            dout = (double *)bout.p;
        }
        LcDecParams DP;
        DP.payload = (const uint32_t *)bpay.p;
        DP.bits = payload_bits;
        DP.T = T;
        DP.sorted = sorted;
        DP.nseg = 0; DP.nblk = 0; DP.seg_bits = 0; DP.nwords = words;
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 8), st));
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 9), st));
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 6), st));
        const unsigned long long ngroups = (n_sync + 31) / 32;
        const unsigned long long want = (ngroups + LC_V3_TPB / 32 - 1) / (LC_V3_TPB / 32);
        int occ = 1;
        LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_dec_v3_kernel, LC_V3_TPB, lc_dec_v3_smem()));
        const unsigned long long cap = (unsigned long long)(occ > 0 ? occ : 1) * lc_sm_count(ctx);
        (void)want;
        const int g = (int)(ngroups < cap ? (ngroups > 0 ? ngroups : 1) : cap);   // one resident wave when there is work for it
        lc_dec_v3_kernel<<<g, LC_V3_TPB, lc_dec_v3_smem(), st>>>(DP, dsync, dstart, desc, n_sync, m, first_value,
                                                                2.0 * eb_abs, (const double *)beval.p,
                                                                (const unsigned long long *)beidx.p, n_esc, dout, dfin);
        { int _rc = lc_debug_check(ctx, "lc_dec_v3_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 1);
        LC_CUDA_OK(cudaMemcpyAsync(hfin, dfin, sizeof(LcV3Final), cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 7), st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        lc_set_kind(ctx, 2);
        if (hfin->status) return hfin->status;
        const int64_t used = hfin->esc_flags[0] ? -1 : (int64_t)hfin->esc_total;
        if (esc_used) *esc_used = used;
        if (used < 0 || (uint64_t)used != n_esc) return 4;
        if (n_esc && hfin->esc_flags[1]) return 5;
        if (!out_on_device) LC_CUDA_OK(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaEventRecord(lc_ev(ctx, 1), st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        return 0;
    }
    if (sync) {                                         // v2: decode straight from the sync table
        LC_CUDA_OK(lc_reserve(baux, 256));
        int *status = (int *)((char *)baux.p + 64);
        int *esc_flags_v2 = (int *)((char *)baux.p + 80);
        (void)esc_flags_v2;
        LC_CUDA_OK(lc_reserve(bsync, n_sync * 8 + 64));
        LC_CUDA_OK(cudaMemcpyAsync(bsync.p, sync, n_sync * 8,
                                   inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        LC_CUDA_OK(cudaMemsetAsync(status, 0, 4, st));
        LcDecParams DP;
        DP.payload = (const uint32_t *)bpay.p;
        DP.bits = payload_bits;
        DP.T = T;
        DP.sorted = sorted;
        DP.nseg = 0; DP.nblk = 0; DP.seg_bits = 0; DP.nwords = words;
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 8), st));
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 9), st));
        const int g = (int)((n_sync + 255) / 256 < (uint64_t)(8 * lc_sm_count(ctx)) ? (n_sync + 255) / 256
                                                                                    : 8 * lc_sm_count(ctx));
        if (code_bytes == 2)
            lc_dec_v2_kernel<uint16_t><<<g, 256, 0, st>>>(DP, (const unsigned long long *)bsync.p, n_sync, bcodes.p, m, status);
        else
            lc_dec_v2_kernel<uint32_t><<<g, 256, 0, st>>>(DP, (const unsigned long long *)bsync.p, n_sync, bcodes.p, m, status);
        { int _rc = lc_debug_check(ctx, "lc_dec_v2_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 1);
        int hit;                                         // the status is checked with the final readback
        return lc_reconstruct(ctx, n, eb_abs, first_value, esc_val, n_esc, out, out_on_device, esc_used,
                              bcodes.p, code_bytes, status, nullptr, &hit);
    }
    // segment size: ~40 average codewords (canonical codes resynchronise
    // within a few codewords), 128..1024 bits, while keeping >= 2 waves of CTAs
    int sub = 2;                                         // 64-bit sub-segments
    {
        const double bps = (double)payload_bits / (double)m;
        while (sub < 16 && 64.0 * sub < 40.0 * bps &&
               (payload_bits / (128ull * sub)) >= (unsigned long long)(2 * 256 * lc_sm_count(ctx)))
            sub *= 2;
    }
    const int seg_bits = 64 * sub;
    const unsigned long long nseg = (payload_bits + seg_bits - 1) / seg_bits + 1;
    const long long nblk = (long long)((nseg + LC_DEC_TPB - 1) / LC_DEC_TPB);
    const unsigned long long scan_tiles = (nseg + LC_TPB * 8 - 1) / (LC_TPB * 8);
    LC_CUDA_OK(lc_reserve(bsync, nseg * sizeof(LcSeg) + 2 * nblk * sizeof(LcBlkOut) + nseg * 8
                                 + scan_tiles * sizeof(LcScanDesc) + 64));
    LcSeg *segs = (LcSeg *)bsync.p;
    LcBlkOut *bo_a = (LcBlkOut *)(segs + nseg), *bo_b = bo_a + nblk;
    unsigned long long *offs = (unsigned long long *)(bo_b + nblk);
    LcScanDesc *sdesc = (LcScanDesc *)(offs + nseg);
    LC_CUDA_OK(lc_reserve(baux, 256));
    int *changed = (int *)baux.p;
    unsigned long long *tot = (unsigned long long *)((char *)baux.p + 16);
    unsigned long long *endpos = (unsigned long long *)((char *)baux.p + 48);
    int *status = (int *)((char *)baux.p + 64);
    int *esc_flags = (int *)((char *)baux.p + 80);
    unsigned int *scan_counter = (unsigned int *)((char *)baux.p + 128);
    LcDecParams DP;
    DP.payload = (const uint32_t *)bpay.p;
    DP.bits = payload_bits;
    DP.T = T;
    DP.sorted = sorted;
    DP.nseg = nseg;
    DP.nblk = nblk;
    DP.seg_bits = seg_bits;
    DP.nwords = words;
    const size_t ssm = lc_dec_stage_bytes(sub);
    // one resident wave: the CTAs stride over the payload ranges, so a grid
    // larger than what fits leaves its late CTAs running at partial occupancy
    int *s_occ = lc_dec_state(ctx);                 // [0..16] per-context (per-device) cache
    if (!s_occ[sub]) {
        int occ = 0;
        switch (sub) {
        case 2: LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_dec_sync_kernel<2>, LC_DEC_TPB, ssm)); break;
        case 4: LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_dec_sync_kernel<4>, LC_DEC_TPB, ssm)); break;
        case 8: LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_dec_sync_kernel<8>, LC_DEC_TPB, ssm)); break;
        default: LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_dec_sync_kernel<16>, LC_DEC_TPB, ssm)); break;
        }
        s_occ[sub] = occ > 0 ? occ : 1;
    }
    const long long pmax = (long long)s_occ[sub] * lc_sm_count(ctx);
    const int pgrid_ = (int)(nblk < pmax ? nblk : pmax);
    auto sync_launch = [&](LcBlkOut *bp, LcBlkOut *bc, int first, int *chg, const int *need) {
        switch (sub) {
        case 2: lc_dec_sync_kernel<2><<<pgrid_, LC_DEC_TPB, ssm, st>>>(DP, segs, bp, bc, first, chg, need); break;
        case 4: lc_dec_sync_kernel<4><<<pgrid_, LC_DEC_TPB, ssm, st>>>(DP, segs, bp, bc, first, chg, need); break;
        case 8: lc_dec_sync_kernel<8><<<pgrid_, LC_DEC_TPB, ssm, st>>>(DP, segs, bp, bc, first, chg, need); break;
        default: lc_dec_sync_kernel<16><<<pgrid_, LC_DEC_TPB, ssm, st>>>(DP, segs, bp, bc, first, chg, need); break;
        }
    };
    int *hchanged = (int *)lc_pinned(ctx);
    sync_launch(bo_b, bo_a, 1, changed, nullptr);
    { int _rc = lc_debug_check(ctx, "lc_dec_sync_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    lc_count_launch(ctx, 1);
    LcBlkOut *bprev = bo_a, *bcur = bo_b;
    int *changed2 = changed + 1;
    // CTA-boundary fix; a cascade (a CTA's own exit moved) needs general passes.
    // That is rare, so the rest of the decode and the reconstruction are queued
    // right behind the fix and the flag is read with their final readback; on a
    // cascade the reconstruction kernels exit at once and the host redoes them.
    // One general pass is queued speculatively: it returns at once unless the
    // fix flagged a cascade (common at high bits per symbol); a second cascade
    // (its own flag) is left to the host.
    LC_CUDA_OK(cudaMemsetAsync(changed, 0, 8, st));
    if (nblk > 1) {
        lc_dec_fix_kernel<<<(int)((nblk - 1 + 127) / 128), 128, 0, st>>>(DP, segs, bo_a, changed);
        { int _rc = lc_debug_check(ctx, "lc_dec_fix_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        sync_launch(bprev, bcur, 0, changed2, changed);
        { int _rc = lc_debug_check(ctx, "lc_dec_sync_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 2);
        LcBlkOut *tmp = bprev; bprev = bcur; bcur = tmp;
    }
    auto tail = [&]() -> int {                           // count scan, write, status
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 8), st));
        LC_CUDA_OK(cudaMemsetAsync(sdesc, 0, scan_tiles * sizeof(LcScanDesc), st));
        LC_CUDA_OK(cudaMemsetAsync(scan_counter, 0, 4, st));
        LC_CUDA_OK(cudaMemsetAsync(tot + 1, 0xff, 8, st));
        {
            const int g = (int)(scan_tiles < (unsigned long long)(2 * lc_sm_count(ctx)) ? scan_tiles : 2 * lc_sm_count(ctx));
            lc_dec_scan_kernel<<<g, LC_TPB, 0, st>>>(segs, nseg, offs, sdesc, scan_counter, tot);
            { int _rc = lc_debug_check(ctx, "lc_dec_scan_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        }
        LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 9), st));
        LC_CUDA_OK(cudaMemsetAsync(endpos, 0xff, 8, st));
        {
            // output window per warp: the typical 32-segment range (+25%), <= 4096 symbols
            const double syms_per_seg = (double)m * seg_bits / (double)(payload_bits ? payload_bits : 1);
            long long cap = (long long)(1.25 * 32.0 * syms_per_seg);
            cap = (cap + 63) / 64 * 64;
            if (cap < 256) cap = 256;
            if (cap > 4096) cap = 4096;
            const size_t wsm = lc_dec_write_smem((int)cap, code_bytes, seg_bits);
            const int wgrid = (int)(nblk < (long long)(2 * lc_sm_count(ctx)) ? nblk : 2 * lc_sm_count(ctx));
            if (code_bytes == 2) {
                lc_dec_write_kernel<uint16_t><<<wgrid, LC_DEC_TPB, wsm, st>>>(DP, segs, offs, bcodes.p, m, endpos, (int)cap);
            } else {
                lc_dec_write_kernel<uint32_t><<<wgrid, LC_DEC_TPB, wsm, st>>>(DP, segs, offs, bcodes.p, m, endpos, (int)cap);
            }
        }
        lc_dec_status_kernel<<<1, 1, 0, st>>>(segs, offs, tot, endpos, m, payload_bits, status);
        { int _rc = lc_debug_check(ctx, "lc_dec_status_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 3);
        return 0;
    };
    { int _rc = tail(); if (_rc) return _rc; }
    int hit = 0;
    int rc = lc_reconstruct(ctx, n, eb_abs, first_value, esc_val, n_esc, out, out_on_device, esc_used, bcodes.p,
                            code_bytes, status, nblk > 1 ? changed2 : nullptr, &hit);
    if (rc != LC_RC_CASCADE) return rc;
    for (int it = 0; it < 1000000; ++it) {              // general passes until no CTA exit moves
        LC_CUDA_OK(cudaMemsetAsync(changed, 0, 4, st));
        sync_launch(bprev, bcur, 0, changed, nullptr);
        { int _rc = lc_debug_check(ctx, "lc_dec_sync_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 1);
        LcBlkOut *tmp = bprev; bprev = bcur; bcur = tmp;
        LC_CUDA_OK(cudaMemcpyAsync(hchanged, changed, 4, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        if (!*hchanged) break;
    }
    { int _rc = tail(); if (_rc) return _rc; }
    return lc_reconstruct(ctx, n, eb_abs, first_value, esc_val, n_esc, out, out_on_device, esc_used, bcodes.p,
                          code_bytes, status, nullptr, &hit);
}

// Reconstruction from decoded codes (compressor.py:358-376, 430-439): exact
// chunked chain + escape checks; inputs already staged in the context.
// Everything the host needs after the reconstruction, packed by one thread so a
// single copy + sync ends the call.
struct LcRecFinal {
    unsigned long long first_bad;
    int esc_flags[2];
    long long cnt_a, cnt_b;     // escapes: state at the last tile start + that tile's aggregate
    int abort_a, abort_b;
};

__global__ void lc_rec_final_kernel(LcRecParams P, LcRecSplit S, long long last, LcRecFinal *f)
{
    f->first_bad = *P.first_bad;
    f->esc_flags[0] = P.esc_flags[0];
    f->esc_flags[1] = P.esc_flags[1];
    f->cnt_a = S.tile_in[last].cnt;
    f->cnt_b = S.tile_seg[last].cnt;
    f->abort_a = P.abort_a ? *P.abort_a : 0;
    f->abort_b = P.abort_b ? *P.abort_b : 0;
}

// Sequential exact reconstruction from chunk first_chunk (the reference loop,
// compressor.py:358-376, on one thread): the decoder's fallback when chunk
// predictions keep failing (more than LC_OPT_MAX_REC relaunches).  Writes the
// escape count the same way the split passes report it.
template <int CB>
__global__ void lc_rec_serial_kernel(LcRecParams P, LcRecFinal *f)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double r = P.anchor_val;
    long long e = P.anchor_cnt;
    for (uint64_t i = (uint64_t)P.first_chunk * LC_L + 1; i < P.n; ++i) {
        const uint32_t code = CB == 2 ? (uint32_t)reinterpret_cast<const uint16_t *>(P.codes)[i - 1]
                                      : reinterpret_cast<const uint32_t *>(P.codes)[i - 1];
        if (code == 0) {                                       // compressor.py:365-369
            if (e < (long long)P.n_esc) {
                r = P.esc_val[e];
                if (P.esc_idx[e] != (unsigned long long)i) P.esc_flags[1] = 1;
            } else {
                P.esc_flags[0] = 1;
            }
            ++e;
        } else {                                               // :370-374
            const int mm = lc_code_m_nz(code);
            if (mm != 0) r = LC_ADD(r, LC_MUL((double)mm, P.delta));
        }
        P.out[i] = r;
    }
    f->first_bad = ~0ULL;
    f->esc_flags[0] = P.esc_flags[0];
    f->esc_flags[1] = P.esc_flags[1];
    f->cnt_a = e;
    f->cnt_b = 0;
    f->abort_a = P.abort_a ? *P.abort_a : 0;
    f->abort_b = P.abort_b ? *P.abort_b : 0;
}

static int lc_reconstruct(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const double *esc_val_in,
                          uint64_t n_esc, double *out, int out_on_device, int64_t *esc_used, void *codes,
                          int code_bytes, const int *abort_a, const int *abort_b, int *abort_hit)
{
    (void)esc_val_in;
    cudaStream_t st = lc_stream(ctx);
    LcBuf *B = lc_dec_bufs(ctx);
    LcBuf &beidx = B[2], &beval = B[3], &bout = B[4], &baux = B[8], &baux2 = B[9];
    const uint64_t m = n - 1;
    int *esc_flags = (int *)((char *)baux.p + 80);
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 6), st));
    double *dout = out;
    if (!out_on_device) {
        LC_CUDA_OK(lc_reserve(bout, n * 8));
        dout = (double *)bout.p;
    }
    const int64_t nchunks = (int64_t)((m + LC_L - 1) / LC_L);
    const int64_t ntiles = (nchunks + LC_TPB - 1) / LC_TPB;
    LC_CUDA_OK(lc_reserve(baux2, LC_MAPSCAN_SCRATCH + 16 + (size_t)(ntiles + 1) * (2 * sizeof(LcSegScan) + sizeof(LcSegDesc) + sizeof(OffMap) + sizeof(double))
                                 + (size_t)nchunks * (16 + sizeof(int) + 5 * sizeof(double)) + 256));
    LcRecParams R;
    R.codes = codes;
    R.code_bytes = code_bytes;
    R.n = n;
    R.delta = 2.0 * eb_abs;
    R.first_value = first_value;
    R.esc_val = (const double *)beval.p;
    R.esc_idx = (const unsigned long long *)beidx.p;
    R.n_esc = n_esc;
    R.first_chunk = 0;
    R.anchor_val = first_value;
    R.anchor_cnt = 0;
    R.nchunks = nchunks;
    R.out = dout;
    R.first_bad = (unsigned long long *)((char *)baux.p + 112);
    R.esc_flags = esc_flags;
    R.abort_a = abort_a;
    R.abort_b = abort_b;
    R.inject_chunk = lc_opt(ctx, LC_OPT_INJECT_REC);
    LcRecFinal *dfin = (LcRecFinal *)((char *)baux.p + 160);
    LcRecFinal *hfin = (LcRecFinal *)((char *)lc_pinned(ctx) + 256);
    *abort_hit = 0;
    LcRecSplit RS;
    void *mapscan_scratch;
    {
        char *pp = (char *)baux2.p;
        RS.tile_seg = (LcSegScan *)pp;           pp += (ntiles + 1) * sizeof(LcSegScan);
        RS.tile_in = (LcSegScan *)pp;            pp += (ntiles + 1) * sizeof(LcSegScan);
        RS.tile_ctr = (unsigned long long *)pp;  pp += 16;
        RS.seg_desc = (LcSegDesc *)pp;           pp += (ntiles + 1) * sizeof(LcSegDesc);
        RS.tile_agg = (OffMap *)pp;              pp += (ntiles + 1) * sizeof(OffMap);
        mapscan_scratch = (void *)pp;            pp += LC_MAPSCAN_SCRATCH;
        RS.tile_D = (double *)pp;                pp += (ntiles + 1) * sizeof(double);
        R.bad_end = (double *)pp;                pp += nchunks * sizeof(double);
        R.chunk_esc = (long long *)pp;           pp += nchunks * sizeof(long long);
        RS.pred.B = (double *)pp;                pp += nchunks * sizeof(double);
        RS.pred.t0 = (double *)pp;               pp += nchunks * sizeof(double);
        RS.pred.t1 = (double *)pp;               pp += nchunks * sizeof(double);
        RS.pred.y = (double *)pp;                pp += nchunks * sizeof(double);
        RS.pred.g0 = (double *)pp;               pp += nchunks * sizeof(double);
        RS.pred.kind = (int *)pp;
    }
    LC_CUDA_OK(cudaMemsetAsync(esc_flags, 0, 8, st));
    lc_set_first_kernel<<<1, 1, 0, st>>>(dout, first_value);
    lc_count_launch(ctx, 1);
    int relaunches = 0;
    lc_dec_state(ctx)[30] = 0;
    for (;;) {
        R.ntiles = (nchunks - R.first_chunk + LC_TPB - 1) / LC_TPB;
        LC_CUDA_OK(cudaMemsetAsync(R.first_bad, 0xff, 8, st));
        // RA look-back state: tile counter and descriptor statuses (contiguous)
        LC_CUDA_OK(cudaMemsetAsync(RS.tile_ctr, 0, 16 + (size_t)R.ntiles * sizeof(LcSegDesc), st));
        lc_rec_a_kernel<<<(int)(R.ntiles < 4 * lc_sm_count(ctx) ? R.ntiles : 4 * lc_sm_count(ctx)), LC_TPB,
                          lc_rec_a_smem_bytes(), st>>>(R, RS);
        { int _rc = lc_debug_check(ctx, "lc_rec_a_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        LC_CUDA_OK((cudaError_t)lc_launch_map_scan(RS.tile_agg, RS.tile_D, R.ntiles, mapscan_scratch, lc_sm_count(ctx), st));
        const int grid_b = (int)(R.ntiles < 3 * lc_sm_count(ctx) ? R.ntiles : 3 * lc_sm_count(ctx));
        if (code_bytes == 2) lc_rec_b_kernel<2><<<grid_b, LC_TPB, lc_rec_b_smem_bytes(), st>>>(R, RS);
        else lc_rec_b_kernel<4><<<grid_b, LC_TPB, lc_rec_b_smem_bytes(), st>>>(R, RS);
        { int _rc = lc_debug_check(ctx, "lc_rec_b_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_rec_final_kernel<<<1, 1, 0, st>>>(R, RS, R.ntiles - 1, dfin);
        lc_count_launch(ctx, 4);
        LC_CUDA_OK(cudaMemcpyAsync(hfin, dfin, sizeof(LcRecFinal), cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        if (hfin->abort_a || hfin->abort_b) {            // the decode failed or needs another pass
            *abort_hit = hfin->abort_b ? LC_RC_CASCADE : hfin->abort_a;   // a cascade voids the status
            return *abort_hit;
        }
        if (hfin->first_bad == ~0ULL) break;
        const unsigned long long fb = hfin->first_bad;
        ++relaunches;
        double anchor;
        long long acnt;
        LC_CUDA_OK(cudaMemcpy(&anchor, R.bad_end + (fb - 1), 8, cudaMemcpyDeviceToHost));
        LC_CUDA_OK(cudaMemcpy(&acnt, R.chunk_esc + fb, 8, cudaMemcpyDeviceToHost));
        R.first_chunk = (int64_t)fb;
        R.anchor_val = anchor;
        R.anchor_cnt = acnt;
        if (relaunches > lc_opt(ctx, LC_OPT_MAX_REC)) {
            // chunk predictions keep failing: finish with the exact sequential chain
            if (code_bytes == 2) lc_rec_serial_kernel<2><<<1, 32, 0, st>>>(R, dfin);
            else lc_rec_serial_kernel<4><<<1, 32, 0, st>>>(R, dfin);
            { int _rc = lc_debug_check(ctx, "lc_rec_serial_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
            lc_count_launch(ctx, 1);
            LC_CUDA_OK(cudaMemcpyAsync(hfin, dfin, sizeof(LcRecFinal), cudaMemcpyDeviceToHost, st));
            LC_CUDA_OK(cudaStreamSynchronize(st));
            lc_dec_state(ctx)[30] = 1;                   // serial path taken (lc_ctx_get_stat)
            break;
        }
    }
    lc_dec_state(ctx)[31] = relaunches;                  // relaunches of the last decompress
    // escape checks (compressor.py:435-439)
    const int hflags[2] = {hfin->esc_flags[0], hfin->esc_flags[1]};
    const long long total_esc = hfin->cnt_a + hfin->cnt_b;
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 7), st));
    lc_set_kind(ctx, 2);
    int64_t used = hflags[0] ? -1 : total_esc;
    if (esc_used) *esc_used = used;
    if (used < 0 || (uint64_t)used != n_esc) return 4;
    if (n_esc && hflags[1]) return 5;
    if (!out_on_device)
        LC_CUDA_OK(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, st));
    LC_CUDA_OK(cudaEventRecord(lc_ev(ctx, 1), st));
    LC_CUDA_OK(cudaStreamSynchronize(st));
    return 0;
}

// Dynamic shared-memory ceilings of the decoder kernels, set once per device
// (lc_ctx_create) to the largest size any call can request.  Calls never
// change them, so concurrent decodes on other host threads cannot race a
// smaller ceiling in between another thread's set and launch.
int lc_decode_init_attrs()
{
    const int wmax16 = (int)lc_dec_write_smem(4096, 2, 64 * 16), wmax32 = (int)lc_dec_write_smem(4096, 4, 64 * 16);
    cudaError_t e = cudaSuccess;
    auto set = [&](const void *f, size_t bytes) {
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    };
    set((const void *)lc_dec_tables_kernel<true>, (LC_DEC_LEN_SMEM + 15) / 16 * 16);
    set((const void *)lc_dec_sync_kernel<2>, lc_dec_stage_bytes(2));
    set((const void *)lc_dec_sync_kernel<4>, lc_dec_stage_bytes(4));
    set((const void *)lc_dec_sync_kernel<8>, lc_dec_stage_bytes(8));
    set((const void *)lc_dec_sync_kernel<16>, lc_dec_stage_bytes(16));
    set((const void *)lc_dec_write_kernel<uint16_t>, wmax16);
    set((const void *)lc_dec_write_kernel<uint32_t>, wmax32);
    set((const void *)lc_rec_a_kernel, lc_rec_a_smem_bytes());
    set((const void *)lc_dec_v3_kernel, lc_dec_v3_smem());
    set((const void *)lc_rec_b_kernel<2>, lc_rec_b_smem_bytes());
    set((const void *)lc_rec_b_kernel<4>, lc_rec_b_smem_bytes());
    return (int)e;
}
