// lc_decode.cu -- chunk-parallel canonical Huffman decode and exact-chain
// reconstruction (sm_100a).
//
// Replaces huffman.decode/_decode_tables/_decode_kernel (huffman.py:75-93,
// 110-132, 153-172) and _decompress_kernel + the escape checks of
// compressor.decompress (compressor.py:358-376, 420-440).
//
// Huffman decode of a v1 (LCKP0001) bitstream, which has no sync points:
//   * the bitstream is cut into S-bit segments, one thread each;
//   * sync passes: each segment decodes from its predecessor's exit position
//     (initially its own start) until it crosses its end; passes repeat until
//     no exit moves (canonical codes resynchronise within a few codewords);
//   * counts are scanned to output offsets and a final pass writes symbols;
//   * the first decoding anomaly on the true path reproduces the reference
//     status (1 invalid codeword, 2 exhausted, 3 trailing bits).
// Reconstruction runs the same chunked exact chain as the encoder
// (lc_chain.cuh): guesses from the m-prefix since the last escape, offset
// maps + look-back, exact re-run, end/start checks (host relaunch on failure).
#include <cub/block/block_scan.cuh>
#include "lc_kernels.cuh"
#include "../../include/lossyckpt_b200.h"

#define LC_SEG_BITS 1024
#define LC_LUT_BITS 12

struct LcDecTables {
    int max_len;
    int used;
    int status;                      // 0 ok, 1 unsupported (max_len > 64)
    int pad;
    unsigned long long first_code[66];
    unsigned long long count[66];
    unsigned long long offset[66];
    unsigned int lut[1 << LC_LUT_BITS];  // (len << 24) | sym; ~0 = no code of length <= LUT_BITS
};

// lengths[nl] -> tables + sorted symbols (canonical order)
__global__ void __launch_bounds__(1024) lc_dec_tables_kernel(const uint8_t *__restrict__ lengths, uint32_t nl,
                                                            LcDecTables *__restrict__ T,
                                                            uint32_t *__restrict__ sorted)
{
    __shared__ int s_cnt[66];
    __shared__ int s_wcnt[32][66];
    __shared__ int s_max;
    __shared__ unsigned long long s_first[66], s_off[66];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    if (tid < 66) s_cnt[tid] = 0;
    if (tid == 0) s_max = 0;
    for (int i = tid; i < 32 * 66; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
    for (int i = tid; i < (1 << LC_LUT_BITS); i += blockDim.x) T->lut[i] = 0xffffffffu;
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
    }
    __syncthreads();
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
            const unsigned long long cw = s_first[l] + rank;
            // shortest length wins on a shared prefix (the reference tries
            // lengths in increasing order); codes that overflow l bits never match
            if (l <= LC_LUT_BITS && cw < (1ULL << l)) {
                const uint32_t lo = (uint32_t)(cw << (LC_LUT_BITS - l));
                const uint32_t nfill = 1u << (LC_LUT_BITS - l);
                for (uint32_t f = 0; f < nfill; ++f) atomicMin(&T->lut[lo + f], ((uint32_t)l << 24) | s);
            }
        }
        __syncwarp();
        if (l > 0 && l <= 64 && (int)(__ffs(peers) - 1) == lane) s_wcnt[wid][l] += __popc(peers);
        __syncwarp();
    }
}

// 64 bits of the MSB-first stream starting at bit p (payload padded by >= 16 bytes)
__device__ __forceinline__ unsigned long long lc_peek64(const uint32_t *__restrict__ w, unsigned long long p)
{
    const unsigned long long wi = p >> 5;
    const int sh = (int)(p & 31);
    const unsigned long long a = __byte_perm(__ldg(w + wi), 0, 0x0123);
    const unsigned long long b = __byte_perm(__ldg(w + wi + 1), 0, 0x0123);
    const unsigned long long hi = (a << 32) | b;
    if (!sh) return hi;
    const unsigned long long c = __byte_perm(__ldg(w + wi + 2), 0, 0x0123);
    return (hi << sh) | (c >> (32 - sh));
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

#define LC_SYNC_K 16

// Per-segment decode state.  bnd[] holds the first codeword starts (bit
// offsets from the segment base) of the last full decode: a later re-decode
// from a different start that lands on one of them is synchronised.
struct __align__(16) LcSeg {
    unsigned long long start;   // bit where this segment's first codeword starts (~0: dead)
    unsigned long long exit;    // first codeword start >= segment end (or stop point)
    unsigned int count;         // codewords started in [start, exit)
    int term;                   // 0 none, 1 invalid, 2 exhausted, 4 clean end at bit_length, 8 dead
    unsigned short bnd[LC_SYNC_K];
    int nbnd;
    unsigned int full_count;    // codewords of the full decode that recorded bnd[] (from bnd[0])
};

struct LcDecParams {
    const uint32_t *payload;    // words (big-endian bit order inside bytes), padded
    unsigned long long bits;    // bit_length
    const LcDecTables *T;
    const uint32_t *sorted;
    unsigned long long nseg;
};

// MSB-first bit reader: the top nb bits of buf are valid (nb in (32, 64] after refill).
struct LcBitReader {
    const uint32_t *w;
    unsigned long long buf, pos, next;
    int nb;
    __device__ __forceinline__ void init(const uint32_t *words, unsigned long long p)
    {
        w = words;
        pos = p;
        const unsigned long long wi = p >> 5;
        const int sh = (int)(p & 31);
        const unsigned long long a = __byte_perm(__ldg(w + wi), 0, 0x0123);
        const unsigned long long b = __byte_perm(__ldg(w + wi + 1), 0, 0x0123);
        buf = ((a << 32) | b) << sh;
        nb = 64 - sh;
        next = wi + 2;
        if (nb <= 32) refill();
    }
    __device__ __forceinline__ void refill()
    {
        buf |= (unsigned long long)__byte_perm(__ldg(w + next), 0, 0x0123) << (32 - nb);
        ++next;
        nb += 32;
    }
    __device__ __forceinline__ void consume(int l)
    {
        if (l >= nb) { init(w, pos + l); return; }   // only for codes longer than the buffer
        buf <<= l;
        nb -= l;
        pos += l;
        if (nb <= 32) refill();
    }
    __device__ __forceinline__ unsigned long long window(int max_len) const
    {
        return max_len > nb ? lc_peek64(w, pos) : buf;
    }
};

// One codeword at the reader; returns its length, 0 for "no codeword within
// max_len bits"; sets *term for anomalies exactly like huffman.py:114-129.
__device__ __forceinline__ int lc_next_symbol(const LcDecParams &P, const LcDecTables &T, int max_len,
                                              const LcBitReader &br, uint32_t *sym, int *term)
{
    if (br.pos >= P.bits) { *term = 4; return 0; }
    const unsigned long long remaining = P.bits - br.pos;
    const int l = lc_decode_one(T, P.sorted, br.window(max_len), max_len, sym);
    if (l == 0) { *term = remaining > (unsigned long long)max_len ? 1 : 2; return 0; }
    if ((unsigned long long)l > remaining) { *term = 2; return 0; }
    return l;
}

// Full decode of [start, seg_end): records boundaries, count, exit, anomaly.
__device__ void lc_walk_full(const LcDecParams &P, const LcDecTables &T, int max_len, unsigned long long start,
                             unsigned long long seg_base, unsigned long long seg_end, LcSeg &S)
{
    LcBitReader br;
    br.init(P.payload, start);
    unsigned int cnt = 0;
    int term = 0, nb = 0;
    while (br.pos < seg_end) {
        uint32_t sym;
        const int l = lc_next_symbol(P, T, max_len, br, &sym, &term);
        if (!l) break;
        if (nb < LC_SYNC_K) S.bnd[nb++] = (unsigned short)(br.pos - seg_base);
        br.consume(l);
        ++cnt;
    }
    S.start = start;
    S.exit = br.pos;
    S.count = cnt;
    S.full_count = cnt;
    S.term = term;
    S.nbnd = nb;
}

// Re-decode from a new start; stops as soon as it lands on a boundary of the
// previous full decode (the remainder is then identical).
__device__ void lc_walk_resync(const LcDecParams &P, const LcDecTables &T, int max_len, unsigned long long start,
                               unsigned long long seg_base, unsigned long long seg_end, LcSeg &S)
{
    LcBitReader br;
    br.init(P.payload, start);
    unsigned int n_new = 0;
    int j = 0;
    while (br.pos < seg_end) {
        while (j < S.nbnd && seg_base + S.bnd[j] < br.pos) ++j;
        if (j < S.nbnd && seg_base + S.bnd[j] == br.pos) {      // synchronised
            S.count = n_new + (S.full_count - (unsigned int)j);
            S.start = start;
            return;
        }
        if (j >= S.nbnd && S.nbnd < LC_SYNC_K) break;            // old decode ended before here
        uint32_t sym;
        int term = 0;
        const int l = lc_next_symbol(P, T, max_len, br, &sym, &term);
        if (!l) { S.start = start; S.exit = br.pos; S.count = n_new; S.term = term; S.nbnd = 0; return; }
        br.consume(l);
        ++n_new;
    }
    lc_walk_full(P, T, max_len, start, seg_base, seg_end, S);    // no sync: decode afresh
}

__device__ __forceinline__ void lc_load_tables(LcDecTables &Ts, const LcDecTables *T)
{
    for (int i = threadIdx.x; i < (int)(sizeof(LcDecTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(&Ts)[i] = reinterpret_cast<const uint32_t *>(T)[i];
    __syncthreads();
}

__global__ void __launch_bounds__(256) lc_dec_sync_kernel(LcDecParams P, const LcSeg *__restrict__ prev,
                                                         LcSeg *__restrict__ cur, int first_pass,
                                                         int *__restrict__ changed)
{
    __shared__ LcDecTables Ts;
    lc_load_tables(Ts, P.T);
    const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.nseg) return;
    const unsigned long long seg_base = t * LC_SEG_BITS, seg_end = seg_base + LC_SEG_BITS;
    LcSeg S;
    if (first_pass) {
        lc_walk_full(P, Ts, Ts.max_len, seg_base, seg_base, seg_end, S);
        cur[t] = S;
        return;
    }
    S = prev[t];
    unsigned long long start = 0;
    if (t > 0) {
        const LcSeg pp = prev[t - 1];
        start = pp.term ? ~0ULL : pp.exit;       // anomaly / end before here: nothing starts here
    }
    if (start == S.start) { cur[t] = S; return; }
    const unsigned long long old_exit = S.exit;
    const int old_term = S.term;
    if (start == ~0ULL) {
        S.start = ~0ULL; S.exit = ~0ULL; S.count = 0; S.term = 8; S.nbnd = 0;
    } else {
        lc_walk_resync(P, Ts, Ts.max_len, start, seg_base, seg_end, S);
    }
    if (S.exit != old_exit || S.term != old_term) atomicExch(changed, 1);
    cur[t] = S;
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

__global__ void __launch_bounds__(256) lc_dec_write_kernel(LcDecParams P, const LcSeg *__restrict__ seg,
                                                          const unsigned long long *__restrict__ off,
                                                          void *out, int out_bytes, unsigned long long m,
                                                          unsigned long long *__restrict__ end_pos)
{
    __shared__ LcDecTables Ts;
    lc_load_tables(Ts, P.T);
    const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.nseg) return;
    const LcSeg S0 = seg[t];
    if (S0.start == ~0ULL || S0.count == 0) return;
    unsigned long long o = off[t];
    if (o >= m) return;
    const unsigned long long seg_end = (t + 1) * LC_SEG_BITS;
    const int max_len = Ts.max_len;
    LcBitReader br;
    br.init(P.payload, S0.start);
    unsigned int cnt = 0;
    while (br.pos < seg_end && cnt < S0.count && o < m) {
        uint32_t sym;
        int term = 0;
        const int l = lc_next_symbol(P, Ts, max_len, br, &sym, &term);
        if (!l) break;
        if (out_bytes == 2) ((uint16_t *)out)[o] = (uint16_t)sym;
        else ((uint32_t *)out)[o] = sym;
        br.consume(l);
        if (o == m - 1) *end_pos = br.pos;
        ++o;
        ++cnt;
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

struct LcRecDesc {
    int st_seg, st_map;
    long long seg_agg_sum, seg_agg_cnt, seg_inc_sum, seg_inc_cnt;
    int seg_agg_has, seg_inc_has;
    int map_kind, pad;
    double mv, mB, mt0, mt1, my, mog;
    double incl_D;
};

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
    LcRecDesc *desc;
    unsigned int *tile_counter;
    double *out;
    unsigned long long *first_bad;
    double *bad_end;
    long long *chunk_esc;       // escapes up to each chunk's start (inclusive of position cL)
    int *esc_flags;             // [0] more escape codes than values, [1] position mismatch
};

__device__ __forceinline__ int64_t lc_code_m(uint32_t code) { return lc_unzigzag(code); }

// ---------------------------------------------------------------------------
// Split reconstruction (no inter-tile waiting): R0 segmented m-prefix per tile,
// R0 scan, RA guess chains + maps, map scan (lc_map_scan_kernel), RB exact chain.

struct LcRecSplit {
    LcSegScan *tile_seg;      // [ntiles] R0 output (tile aggregate)
    LcSegScan *tile_in;       // [ntiles] R0 scan output (state at each tile start)
    OffMap *tile_agg;         // [ntiles] RA output
    double *tile_D;           // [ntiles + 1] map scan output
    LcChunkPred pred;         // RA -> RB
};

__device__ __forceinline__ void lc_load_codes_tile(const LcRecParams &P, long long pbeg, uint32_t *cs)
{
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
#pragma unroll 8
    for (int k = 0; k < LC_L; ++k) {
        const int off = k * LC_TPB + tid;
        const long long pos = pbeg + off;
        uint32_t v = 0;
        if (pos < nel) v = P.code_bytes == 2 ? (uint32_t)reinterpret_cast<const uint16_t *>(P.codes)[pos]
                                             : reinterpret_cast<const uint32_t *>(P.codes)[pos];
        cs[(off >> 5) * LC_ROW + (off & 31)] = v;
    }
}

__device__ __forceinline__ LcSegScan lc_chunk_segscan(const uint32_t *crow, int len)
{
    LcSegScan mine; mine.sum = 0; mine.cnt = 0; mine.has = 0; mine.moved = 0;
    for (int j = 0; j < len; ++j) {
        const uint32_t code = crow[j];
        if (code == 0) { mine.sum = 0; mine.cnt += 1; mine.has = 1; mine.moved = 0; }
        else { const int64_t mm = lc_code_m(code); mine.sum += mm; mine.moved |= (mm != 0); }
    }
    return mine;
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

__global__ void __launch_bounds__(LC_TPB) lc_rec0_kernel(LcRecParams P, LcRecSplit S)
{
    __shared__ uint32_t cs[LC_TPB * LC_ROW];
    __shared__ LcSegScan wseg[LC_TPB / 32];
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long c = cbeg + tid;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - c * LC_L) : 0;
        __syncthreads();
        lc_load_codes_tile(P, cbeg * LC_L, cs);
        __syncthreads();
        const LcSegScan mine = lc_chunk_segscan(cs + tid * LC_ROW, len);
        LcSegScan agg;
        lc_block_segscan(mine, wseg, &agg);
        if (tid == 0) S.tile_seg[t] = agg;
    }
}

__global__ void __launch_bounds__(1024) lc_rec0_scan_kernel(LcRecSplit S, long long ntiles, long long anchor_cnt)
{
    // sequential runs per thread + block scan of the runs (LcSegScan is a monoid)
    __shared__ LcSegScan wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long per = (ntiles + 1023) / 1024;
    const long long b0 = (long long)tid * per, b1 = min(ntiles, b0 + per);
    LcSegScan run; run.sum = 0; run.cnt = 0; run.has = 0; run.moved = 0;
    for (long long t = b0; t < b1; ++t) run = lc_segscan_op(run, S.tile_seg[t]);
    LcSegScan inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const LcSegScan up = lc_shfl_up_seg(inc, o);
        if (lane >= o) inc = lc_segscan_op(up, inc);
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (tid == 0)
        for (int w = 1; w < 32; ++w) wsum[w] = lc_segscan_op(wsum[w - 1], wsum[w]);
    __syncthreads();
    if (wid > 0) inc = lc_segscan_op(wsum[wid - 1], inc);
    LcSegScan exc = lc_shfl_up_seg(inc, 1);
    if (lane == 0) {
        if (wid > 0) exc = wsum[wid - 1];
        else { exc.sum = 0; exc.cnt = 0; exc.has = 0; exc.moved = 0; }
    }
    LcSegScan st; st.sum = 0; st.cnt = anchor_cnt; st.has = 1; st.moved = 0;   // launch anchor
    st = lc_segscan_op(st, exc);
    for (long long t = b0; t < b1; ++t) {
        S.tile_in[t] = st;
        st = lc_segscan_op(st, S.tile_seg[t]);
    }
}

__global__ void __launch_bounds__(LC_TPB, 2) lc_rec_a_kernel(LcRecParams P, LcRecSplit S)
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    uint32_t *cs = reinterpret_cast<uint32_t *>(lc_dyn_smem);
    __shared__ LcSegScan wseg[LC_TPB / 32];
    __shared__ OffMap warp_agg[LC_TPB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long nel = (long long)P.n - 1;
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long c = cbeg + tid;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - c * LC_L) : 0;
        __syncthreads();
        lc_load_codes_tile(P, cbeg * LC_L, cs);
        __syncthreads();
        const uint32_t *crow = cs + tid * LC_ROW;
        const LcSegScan mine = lc_chunk_segscan(crow, len);
        LcSegScan agg;
        const LcSegScan exc = lc_block_segscan(mine, wseg, &agg);
        const LcSegScan before = lc_segscan_op(S.tile_in[t], exc);
        const LcSegScan after = lc_segscan_op(before, mine);
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
        OffMap H;
        if (len > 0) {
            P.chunk_esc[c] = before.cnt;
            double r = g0;
            long long e = before.cnt;
            LcEvents E;
            lc_events_init(E, g0);
            bool pend = false;
            double pr = 0.0, pc = 0.0, prn = 0.0;
            for (int j = 0; j < len; ++j) {
                const uint32_t code = crow[j];
                const bool esc = code == 0;
                const int64_t m = lc_code_m(code);
                const double inc_ = LC_MUL((double)m, P.delta);
                double rn = m != 0 ? LC_ADD(r, inc_) : r;
                if (esc) { rn = e < (long long)P.n_esc ? P.esc_val[e] : 0.0; ++e; }
                lc_events_step_if(E, pend, j - 1, pr, pc, prn);
                lc_events_escape_if(E, esc);
                pend = !esc && m != 0;
                pr = r; pc = inc_; prn = rn;
                r = rn;
            }
            lc_events_step_if(E, pend, len - 1, pr, pc, prn);
            if (!lc_events_finish(E, g0, H)) {          // events: replay, compose at flagged steps
                double r2 = g0;
                for (int j = 0; j < len; ++j) {
                    const int64_t m = lc_code_m(crow[j]);  // no escape here (E.esc would be set)
                    if (m != 0) {
                        const double inc_ = LC_MUL((double)m, P.delta);
                        const double rn = LC_ADD(r2, inc_);
                        if ((E.mask >> j) & 1u) lc_map_step(H, r2, inc_, rn);
                        r2 = rn;
                    }
                }
            }
            if (c + 1 < P.nchunks) lc_map_shift_out(H, LC_SUB(r, g1));
        } else {
            H = lc_map_neutral();
        }
        OffMap inc_map = H;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const OffMap up = lc_shfl_up_map(inc_map, o);
            if (lane >= o) inc_map = lc_map_compose(inc_map, up);
        }
        if (lane == 31) warp_agg[wid] = inc_map;
        __syncthreads();
        if (tid == 0)
            for (int w = 1; w < LC_TPB / 32; ++w) warp_agg[w] = lc_map_compose(warp_agg[w], warp_agg[w - 1]);
        __syncthreads();
        if (wid > 0) inc_map = lc_map_compose(inc_map, warp_agg[wid - 1]);
        OffMap exc_map = lc_shfl_up_map(inc_map, 1);
        if (lane == 0) exc_map = wid > 0 ? warp_agg[wid - 1] : lc_map_neutral();
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

__global__ void __launch_bounds__(LC_TPB, 2) lc_rec_b_kernel(LcRecParams P, LcRecSplit S)
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    double *ys = reinterpret_cast<double *>(lc_dyn_smem);
    uint32_t *cs = reinterpret_cast<uint32_t *>(ys + LC_TPB * LC_ROW);
    __shared__ double starts[LC_TPB + 1];
    const int tid = threadIdx.x;
    const long long nel = (long long)P.n - 1;
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        const long long cbeg = P.first_chunk + t * LC_TPB;
        const long long pbeg = cbeg * LC_L;
        const long long c = cbeg + tid;
        const long long p0 = c * LC_L;
        const int len = (c < P.nchunks) ? (int)min((long long)LC_L, nel - p0) : 0;
        __syncthreads();
        lc_load_codes_tile(P, pbeg, cs);
        const double Dt = S.tile_D[t];
        double start = 0.0;
        if (len > 0) {
            OffMap m;
            m.kind = S.pred.kind[c]; m.B = S.pred.B[c]; m.t0 = S.pred.t0[c]; m.t1 = S.pred.t1[c]; m.y = S.pred.y[c];
            m.v = 0.0; m.og = 0.0;
            start = lc_apply_offset(S.pred.g0[c], lc_map_eval(m, Dt));
        }
        starts[tid] = start;
        if (tid == LC_TPB - 1) {
            const long long cn = cbeg + LC_TPB;
            starts[LC_TPB] = (cn < P.nchunks) ? lc_apply_offset(S.pred.g0[cn], S.tile_D[t + 1]) : 0.0;
        }
        __syncthreads();
        const uint32_t *crow = cs + tid * LC_ROW;
        double *yrow = ys + tid * LC_ROW;
        if (len > 0) {
            double r = start;
            long long e = P.chunk_esc[c];
            for (int j = 0; j < len; ++j) {
                const uint32_t code = crow[j];
                const int64_t m = lc_code_m(code);
                double rn = m != 0 ? LC_ADD(r, LC_MUL((double)m, P.delta)) : r;   // compressor.py:371-374
                if (code == 0) {                                                   // :365-369
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
            }
            if (c + 1 < P.nchunks && lc_bits(r) != lc_bits(starts[tid + 1])) {
                P.bad_end[c] = r;
                atomicMin(P.first_bad, (unsigned long long)(c + 1));
            }
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < LC_L; ++k) {
            const int off = k * LC_TPB + tid;
            const long long pos = pbeg + 1 + off;
            if (pos <= nel) __stcs(P.out + pos, ys[(off >> 5) * LC_ROW + (off & 31)]);
        }
    }
}

size_t lc_rec_a_smem_bytes() { return sizeof(uint32_t) * LC_TPB * LC_ROW; }
size_t lc_rec_b_smem_bytes() { return sizeof(double) * LC_TPB * LC_ROW + sizeof(uint32_t) * LC_TPB * LC_ROW; }


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

int lc_decompress_impl(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value,
                       const uint8_t *code_lengths, uint64_t n_lengths, const uint8_t *payload,
                       uint64_t payload_bytes, uint64_t payload_bits, const uint64_t *esc_idx,
                       const double *esc_val, uint64_t n_esc, int inputs_on_device, double *out,
                       int out_on_device, int64_t *esc_used)
{
    if (n < 2 || n_lengths == 0 || payload_bits > 8 * payload_bytes) return 12;
    cudaStream_t st = lc_stream(ctx);
    LcBuf *B = lc_dec_bufs(ctx);      // ctx->dec[10]
    LcBuf &bpay = B[0], &blen = B[1], &beidx = B[2], &beval = B[3], &bout = B[4], &bcodes = B[5], &btab = B[6],
          &bsync = B[7], &baux = B[8], &baux2 = B[9];
    LC_CUDA_OK(cudaEventRecord(lc_ev(ctx, 0), st));
    const uint64_t m = n - 1;
    const uint64_t words = (payload_bytes + 3) / 4 + 4;
    LC_CUDA_OK(lc_reserve(bpay, words * 4));
    LC_CUDA_OK(cudaMemsetAsync(bpay.p, 0, words * 4, st));
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
    lc_dec_tables_kernel<<<1, 1024, 0, st>>>((const uint8_t *)blen.p, (uint32_t)n_lengths, T, sorted);
    { int _rc = lc_debug_check(ctx, "lc_dec_tables_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    lc_count_launch(ctx, 2);
    // Huffman decode
    const int code_bytes = n_lengths <= 65536 ? 2 : 4;
    LC_CUDA_OK(lc_reserve(bcodes, m * code_bytes + 16));
    const unsigned long long nseg = (payload_bits + LC_SEG_BITS - 1) / LC_SEG_BITS + 1;
    const unsigned long long scan_tiles = (nseg + LC_TPB * 8 - 1) / (LC_TPB * 8);
    LC_CUDA_OK(lc_reserve(bsync, 2 * nseg * sizeof(LcSeg) + nseg * 8 + scan_tiles * sizeof(LcScanDesc) + 64));
    LcSeg *sa = (LcSeg *)bsync.p, *sb = sa + nseg;
    unsigned long long *offs = (unsigned long long *)(sb + nseg);
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
    const int sblocks = (int)((nseg + 255) / 256);
    int *hchanged = (int *)lc_pinned(ctx);
    lc_dec_sync_kernel<<<sblocks, 256, 0, st>>>(DP, sa, sa, 1, changed);
    { int _rc = lc_debug_check(ctx, "lc_dec_sync_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    lc_count_launch(ctx, 1);
    LcSeg *prev = sa, *cur = sb;
    for (int it = 0; it < 1000000; ++it) {
        LC_CUDA_OK(cudaMemsetAsync(changed, 0, 4, st));
        lc_dec_sync_kernel<<<sblocks, 256, 0, st>>>(DP, prev, cur, 0, changed);
        { int _rc = lc_debug_check(ctx, "lc_dec_sync_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 1);
        LcSeg *tmp = prev; prev = cur; cur = tmp;
        LC_CUDA_OK(cudaMemcpyAsync(hchanged, changed, 4, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        if (!*hchanged) break;
    }
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 8), st));
    LC_CUDA_OK(cudaMemsetAsync(sdesc, 0, scan_tiles * sizeof(LcScanDesc), st));
    LC_CUDA_OK(cudaMemsetAsync(scan_counter, 0, 4, st));
    LC_CUDA_OK(cudaMemsetAsync(tot + 1, 0xff, 8, st));
    {
        const int g = (int)(scan_tiles < (unsigned long long)(2 * lc_sm_count(ctx)) ? scan_tiles : 2 * lc_sm_count(ctx));
        lc_dec_scan_kernel<<<g, LC_TPB, 0, st>>>(prev, nseg, offs, sdesc, scan_counter, tot);
        { int _rc = lc_debug_check(ctx, "lc_dec_scan_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    }
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 9), st));
    LC_CUDA_OK(cudaMemsetAsync(endpos, 0xff, 8, st));
    lc_dec_write_kernel<<<sblocks, 256, 0, st>>>(DP, prev, offs, bcodes.p, code_bytes, m, endpos);
    lc_dec_status_kernel<<<1, 1, 0, st>>>(prev, offs, tot, endpos, m, payload_bits, status);
    { int _rc = lc_debug_check(ctx, "lc_dec_status_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    lc_count_launch(ctx, 3);
    int *hstat = (int *)lc_pinned(ctx);
    LC_CUDA_OK(cudaMemcpyAsync(hstat, status, 4, cudaMemcpyDeviceToHost, st));
    LC_CUDA_OK(cudaStreamSynchronize(st));
    if (*hstat) return *hstat;

    // reconstruction
    LC_CUDA_OK(cudaEventRecord(lc_phase_ev(ctx, 6), st));
    double *dout = out;
    if (!out_on_device) {
        LC_CUDA_OK(lc_reserve(bout, n * 8));
        dout = (double *)bout.p;
    }
    const int64_t nchunks = (int64_t)((m + LC_L - 1) / LC_L);
    const int64_t ntiles = (nchunks + LC_TPB - 1) / LC_TPB;
    LC_CUDA_OK(lc_reserve(baux2, (size_t)(ntiles + 1) * (2 * sizeof(LcSegScan) + sizeof(OffMap) + sizeof(double))
                                 + (size_t)nchunks * (16 + sizeof(int) + 5 * sizeof(double)) + 256));
    LcRecParams R;
    R.codes = bcodes.p;
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
    R.desc = nullptr;
    R.tile_counter = nullptr;
    R.out = dout;
    R.first_bad = (unsigned long long *)((char *)baux.p + 112);
    R.esc_flags = esc_flags;
    LcRecSplit RS;
    {
        char *pp = (char *)baux2.p;
        RS.tile_seg = (LcSegScan *)pp;           pp += (ntiles + 1) * sizeof(LcSegScan);
        RS.tile_in = (LcSegScan *)pp;            pp += (ntiles + 1) * sizeof(LcSegScan);
        RS.tile_agg = (OffMap *)pp;              pp += (ntiles + 1) * sizeof(OffMap);
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
    static bool attr_b = false;
    if (!attr_b) {
        LC_CUDA_OK(cudaFuncSetAttribute(lc_rec_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)lc_rec_a_smem_bytes()));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_rec_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)lc_rec_b_smem_bytes()));
        attr_b = true;
    }
    LC_CUDA_OK(cudaMemsetAsync(esc_flags, 0, 8, st));
    lc_set_first_kernel<<<1, 1, 0, st>>>(dout, first_value);
    lc_count_launch(ctx, 1);
    const int grid_cap = 2 * lc_sm_count(ctx);
    unsigned long long *hbad = (unsigned long long *)lc_pinned(ctx);
    int relaunches = 0;
    for (;;) {
        R.ntiles = (nchunks - R.first_chunk + LC_TPB - 1) / LC_TPB;
        LC_CUDA_OK(cudaMemsetAsync(R.first_bad, 0xff, 8, st));
        const int grid = (int)(R.ntiles < grid_cap ? R.ntiles : grid_cap);
        lc_rec0_kernel<<<(int)(R.ntiles < 3 * grid_cap ? R.ntiles : 3 * grid_cap), LC_TPB, 0, st>>>(R, RS);
        lc_rec0_scan_kernel<<<1, 1024, 0, st>>>(RS, R.ntiles, R.anchor_cnt);
        lc_rec_a_kernel<<<grid, LC_TPB, lc_rec_a_smem_bytes(), st>>>(R, RS);
        { int _rc = lc_debug_check(ctx, "lc_rec_a_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_map_scan_kernel<<<1, 1024, 0, st>>>(RS.tile_agg, RS.tile_D, R.ntiles);
        lc_rec_b_kernel<<<grid, LC_TPB, lc_rec_b_smem_bytes(), st>>>(R, RS);
        { int _rc = lc_debug_check(ctx, "lc_rec_b_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_count_launch(ctx, 5);
        LC_CUDA_OK(cudaMemcpyAsync(hbad, R.first_bad, 8, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        if (*hbad == ~0ULL) break;
        const unsigned long long fb = *hbad;
        ++relaunches;
        double anchor;
        long long acnt;
        LC_CUDA_OK(cudaMemcpy(&anchor, R.bad_end + (fb - 1), 8, cudaMemcpyDeviceToHost));
        LC_CUDA_OK(cudaMemcpy(&acnt, R.chunk_esc + fb, 8, cudaMemcpyDeviceToHost));
        R.first_chunk = (int64_t)fb;
        R.anchor_val = anchor;
        R.anchor_cnt = acnt;
        if (relaunches > 100000) { lc_set_err(ctx, "reconstruction did not converge"); return 20; }
    }
    // escape checks (compressor.py:435-439)
    int hflags[2];
    long long total_esc;
    LC_CUDA_OK(cudaMemcpy(hflags, esc_flags, 8, cudaMemcpyDeviceToHost));
    {
        // total escape codes = state at the last tile start + that tile's aggregate
        LcSegScan a, b;
        LC_CUDA_OK(cudaMemcpy(&a, RS.tile_in + (R.ntiles - 1), sizeof(LcSegScan), cudaMemcpyDeviceToHost));
        LC_CUDA_OK(cudaMemcpy(&b, RS.tile_seg + (R.ntiles - 1), sizeof(LcSegScan), cudaMemcpyDeviceToHost));
        total_esc = a.cnt + b.cnt;
    }
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
