// lc_huff.cu -- on-device canonical Huffman codebook and chunked encoder.
//
// Replaces huffman.code_lengths (huffman.py:21-55), canonical_codes
// (huffman.py:58-72) and encode/_encode_kernel (huffman.py:96-107,135-150).
//
// Codebook (one block, no host step):
//   1. compact used symbols, key = (freq << 32 | symbol)
//   2. sort keys (bitonic, smem when they fit, else global)
//   3. two-queue Huffman merge: leaves in (freq, symbol) order, internal
//      nodes in creation order, a leaf wins ties -- the exact pop order of
//      the reference's heapq over (freq, insertion counter)
//   4. depths (reverse creation order), canonical codes per length
// Encoder: one tile = 256 threads x 32 codes; per-thread bit counts, block
// scan, decoupled look-back on (bits, escapes); words strictly inside a
// thread's bit range are stored directly, the two boundary words use
// atomicOr on a zeroed payload.  Escape positions are compacted in the same
// pass (compressor.py:409-410).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include "lc_kernels.cuh"

#define LC_CB_THREADS 1024
#define LC_CB_SMEM_KEYS 4096
#define LC_ENC_TAB 8192                 // smem code table entries: (len << 27) | code, codes <= 27 bits


__device__ __forceinline__ void lc_bitonic_sort(unsigned long long *a, int npow2)
{
    const int half = npow2 >> 1;
    for (int k = 2; k <= npow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int q = threadIdx.x; q < half; q += blockDim.x) {
                const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));   // lower index of the pair
                const int ixj = i | j;
                const unsigned long long ai = a[i], aj = a[ixj];
                const bool up = (i & k) == 0;
                if ((ai > aj) == up) { a[i] = aj; a[ixj] = ai; }
            }
            __syncthreads();
        }
    }
}

// Large alphabets (more used symbols than fit the shared-memory working set):
// sort the (freq, p) keys with a block radix sort on the frequency (stable, so
// equal frequencies stay in p = symbol order) held in registers, 16 keys per
// thread, instead of a bitonic network over global memory (~100 passes with a
// CTA barrier each).  temp: the (unused) dynamic shared memory.
#define LC_CB_RADIX_ITEMS 16
#define LC_CB_MAXB 2048                 // merge batches recorded for the depth pass
#define LC_CB_RADIX_KEYS (LC_CB_THREADS * LC_CB_RADIX_ITEMS)
static_assert(sizeof(cub::BlockRadixSort<uint32_t, LC_CB_THREADS, LC_CB_RADIX_ITEMS, uint32_t>::TempStorage) <=
                  (2 * sizeof(unsigned long long) + 2 * sizeof(int) + sizeof(uint32_t) + 1) * LC_CB_SMEM_KEYS,
              "radix-sort scratch must fit the codebook's dynamic shared memory");
__device__ __forceinline__ void lc_radix_sort_keys(unsigned long long *keys, int k, int npow2, void *temp)
{
    typedef cub::BlockRadixSort<uint32_t, LC_CB_THREADS, LC_CB_RADIX_ITEMS, uint32_t> RS;
    uint32_t kf[LC_CB_RADIX_ITEMS], kv[LC_CB_RADIX_ITEMS];
#pragma unroll
    for (int i = 0; i < LC_CB_RADIX_ITEMS; ++i) {
        const int idx = threadIdx.x * LC_CB_RADIX_ITEMS + i;
        const unsigned long long key = idx < k ? keys[idx] : ~0ull;
        kf[i] = (uint32_t)(key >> 32);
        kv[i] = (uint32_t)key;
    }
    __syncthreads();
    RS(*reinterpret_cast<typename RS::TempStorage *>(temp)).Sort(kf, kv);
#pragma unroll
    for (int i = 0; i < LC_CB_RADIX_ITEMS; ++i) {
        const int idx = threadIdx.x * LC_CB_RADIX_ITEMS + i;
        if (idx < npow2) keys[idx] = ((unsigned long long)kf[i] << 32) | kv[i];
    }
    __syncthreads();
}

// hist[nbins] -> lengths[nbins], codes[nbins], meta.  Working arrays live in
// shared memory when at most LC_CB_SMEM_KEYS symbols are used (SMEM), else in
// the global scratch (gkeys: 3*nbins u64, ifreq: nbins u64, parent: 2*nbins int).
// Used symbols are numbered p = 0..k-1 in symbol order; sort keys are
// (freq << 32 | p), so (freq, p) order is the reference's (freq, symbol) order.
template <bool SMEM>
__device__ __forceinline__ void lc_codebook_body(const uint32_t *__restrict__ hist, uint32_t nbins,
                                                 uint8_t *__restrict__ lengths, unsigned long long *__restrict__ codes,
                                                 unsigned long long *__restrict__ gkeys,
                                                 unsigned long long *__restrict__ ifreq_g, int *__restrict__ parent_g,
                                                 LcCodebookOut *out, int k, int wbase, uint32_t wsb, uint32_t wse,
                                                 int *s_len_count, int *s_len_start, unsigned long long *s_first,
                                                 unsigned long long *s_bits, int *s_wmax, int (*s_wcnt)[65])
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NWARP = LC_CB_THREADS / 32;
    const int cap = SMEM ? LC_CB_SMEM_KEYS : (int)(2 * nbins);
    unsigned long long *keys = SMEM ? reinterpret_cast<unsigned long long *>(lc_dyn_smem) : gkeys;
    unsigned long long *ifreq = SMEM ? keys + LC_CB_SMEM_KEYS : ifreq_g;
    int *parent = SMEM ? reinterpret_cast<int *>(ifreq + LC_CB_SMEM_KEYS) : parent_g;
    uint32_t *syms = SMEM ? reinterpret_cast<uint32_t *>(parent + 2 * LC_CB_SMEM_KEYS)
                          : reinterpret_cast<uint32_t *>(gkeys + cap);
    uint8_t *lenp = reinterpret_cast<uint8_t *>(syms + (SMEM ? LC_CB_SMEM_KEYS : nbins));
    int npow2 = 1;
    while (npow2 < k) npow2 <<= 1;
    // 1b. compaction in symbol order (warp ranges, ballot ranks)
    int wpos = wbase;
    for (uint32_t s0 = wsb; s0 < wse; s0 += 256) {             // 8 independent loads per lane
        uint32_t hv[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t sy = s0 + 32 * g + lane;
            hv[g] = sy < wse ? __ldg(hist + sy) : 0u;
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t sy = s0 + 32 * g + lane;
            const unsigned bal = __ballot_sync(0xffffffffu, hv[g] != 0);
            if (hv[g]) {
                const int pp = wpos + __popc(bal & ((1u << lane) - 1u));
                keys[pp] = ((unsigned long long)hv[g] << 32) | (uint32_t)pp;
                syms[pp] = sy;
            }
            wpos += __popc(bal);
        }
    }
    for (int i = k + tid; i < npow2; i += LC_CB_THREADS) keys[i] = ~0ULL;
    __syncthreads();
    if (k == 1) {                                   // huffman.py:33-35
        if (tid == 0) {
            const uint32_t sy = syms[0];
            lengths[sy] = 1;
            codes[sy] = 0;
            out->total_bits = keys[0] >> 32;
            out->n_esc = hist[0];
            out->max_len = 1; out->used = 1; out->status = 0;
        }
        return;
    }
    if (tid == 0) out->stamp[0] = lc_gtimer();
    // 2. sort by (freq, symbol)
    if (!SMEM && npow2 <= LC_CB_RADIX_KEYS) lc_radix_sort_keys(keys, k, npow2, lc_dyn_smem);
    else lc_bitonic_sort(keys, npow2);
    if (tid == 0) out->stamp[1] = lc_gtimer();

    // 3. two-queue merge (huffman.py:36-48: heapq pops (freq, counter); leaves were
    //    pushed first, so with leaves sorted by (freq, symbol) and internal nodes in
    //    creation order a leaf wins ties).  Leaves 0..k-1; internal node m has
    //    freq ifreq[m]; parent[leaf] at [0,k), parent[k + m] for internal node m.
    //    Batched: with t the smallest head, every queued item of freq <= 2t is
    //    picked before any node created from them (new nodes are >= 2t and lose
    //    ties to older items), so the batch's picks are the merged order of the
    //    two queues up to 2t and its pairs become new nodes in parallel (merge
    //    path per pair).  t at least doubles per batch: O(log total) batches.
    // batch starts (the first internal node each batch creates): every node's
    // parent is created in a later batch, so depths follow batch by batch in
    // reverse (step 4)
    __shared__ int s_bstart[LC_CB_MAXB + 1];
    __shared__ int s_nbatch;
    {
        __shared__ int s_li, s_ii, s_m, s_na, s_nb, s_go;
        if (tid == 0) { s_li = 0; s_ii = 0; s_m = 0; s_nbatch = 0; }
        __syncthreads();
        const unsigned long long INF = ~0ULL;
        for (;;) {
            if (tid == 0) {
                const int li = s_li, ii = s_ii, m = s_m;
                s_go = m < k - 1;
                if (s_go) {
                    if (s_nbatch <= LC_CB_MAXB) s_bstart[s_nbatch] = m;
                    ++s_nbatch;
                    const unsigned long long lf = li < k ? keys[li] >> 32 : INF;
                    const unsigned long long nf = ii < m ? ifreq[ii] : INF;
                    const unsigned long long t = lf < nf ? lf : nf;
                    const unsigned long long T = t > (INF >> 1) ? INF : 2 * t;
                    int lo = li, hi = k;                          // leaves with freq <= T
                    while (lo < hi) { const int md = (lo + hi) >> 1; if ((keys[md] >> 32) <= T) lo = md + 1; else hi = md; }
                    const int la = lo;
                    lo = ii; hi = m;                              // internal nodes with freq <= T
                    while (lo < hi) { const int md = (lo + hi) >> 1; if (ifreq[md] <= T) lo = md + 1; else hi = md; }
                    s_na = la - li;
                    s_nb = lo - ii;
                    if (s_na + s_nb < 2) {                        // one sequential step
                        int pk[2];
                        unsigned long long f[2];
                        int l2 = li, i2 = ii;
                        for (int q = 0; q < 2; ++q) {
                            const unsigned long long a = l2 < k ? keys[l2] >> 32 : INF;
                            const unsigned long long b = i2 < m ? ifreq[i2] : INF;
                            if (a <= b) { pk[q] = l2; f[q] = a; ++l2; } else { pk[q] = k + i2; f[q] = b; ++i2; }
                        }
                        ifreq[m] = f[0] + f[1];
                        parent[pk[0]] = m;
                        parent[pk[1]] = m;
                        s_li = l2; s_ii = i2; s_m = m + 1;
                        s_na = -1;
                    }
                }
            }
            __syncthreads();
            if (!s_go) break;
            const int li = s_li, ii = s_ii, m = s_m, na = s_na, nb = s_nb;
            if (na >= 0) {
                const int npairs = (na + nb) >> 1;
                // merged position p -> (# leaves among the first p picks); leaf wins ties
                auto split = [&](int p) -> int {
                    int lo = max(0, p - nb), hi = min(p, na);
                    while (lo < hi) {
                        const int i = (lo + hi) >> 1, j = p - i;
                        if ((keys[li + i] >> 32) <= ifreq[ii + j - 1]) lo = i + 1; else hi = i;
                    }
                    return lo;
                };
                auto item = [&](int p, unsigned long long *f) -> int {
                    const int i = split(p), j = p - i;
                    const bool leaf = i < na && (j >= nb || (keys[li + i] >> 32) <= ifreq[ii + j]);
                    if (leaf) { *f = keys[li + i] >> 32; return li + i; }
                    *f = ifreq[ii + j];
                    return k + ii + j;
                };
                for (int q = tid; q < npairs; q += LC_CB_THREADS) {
                    unsigned long long fa, fb;
                    const int a = item(2 * q, &fa), b = item(2 * q + 1, &fb);
                    ifreq[m + q] = fa + fb;                       // beyond the batch's read range
                    parent[a] = m + q;
                    parent[b] = m + q;
                }
                __syncthreads();
                if (tid == 0) {
                    const int used = split(2 * npairs);
                    s_li = li + used;
                    s_ii = ii + 2 * npairs - used;
                    s_m = m + npairs;
                }
            }
            __syncthreads();
        }
    }
    __syncthreads();
    if (tid == 0) out->stamp[2] = lc_gtimer();
    // 4. depths of internal nodes: pointer jumping (root k-2 has depth 0)
    int *D = reinterpret_cast<int *>(ifreq);         // freqs no longer needed
    int *A = D + k;
    const int ni = k - 1;
    constexpr int NJ = 8;
    const int nbatch = s_nbatch;
    if (nbatch <= LC_CB_MAXB && (ni > NJ * LC_CB_THREADS || nbatch < 32)) {
        // reverse batch order: a batch's parents are all in later batches
        if (tid == 0) D[ni - 1] = 0;
        __syncthreads();
        for (int bi = nbatch - 1; bi >= 0; --bi) {
            const int b0 = s_bstart[bi], b1 = bi + 1 < nbatch ? s_bstart[bi + 1] : ni;
            for (int m = b0 + tid; m < b1; m += LC_CB_THREADS)
                if (m != ni - 1) D[m] = D[parent[k + m]] + 1;
            __syncthreads();
        }
    } else if (ni <= NJ * LC_CB_THREADS) {
        for (int m = tid; m < ni; m += LC_CB_THREADS) {
            const bool root = m == ni - 1;
            D[m] = root ? 0 : 1;
            A[m] = root ? -1 : parent[k + m];
        }
        __syncthreads();
        for (int r = 1; r < ni; r <<= 1) {
            int nd[NJ], na[NJ];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int m = tid + j * LC_CB_THREADS;
                nd[j] = 0; na[j] = -1;
                if (m < ni) {
                    const int a = A[m];
                    nd[j] = D[m];
                    if (a >= 0) { nd[j] += D[a]; na[j] = A[a]; }
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int m = tid + j * LC_CB_THREADS;
                if (m < ni) { D[m] = nd[j]; A[m] = na[j]; }
            }
            __syncthreads();
        }
    } else {
        if (tid == 0) {
            D[ni - 1] = 0;
            for (int m = ni - 2; m >= 0; --m) D[m] = D[parent[k + m]] + 1;
        }
        __syncthreads();
    }
    if (tid == 0) out->stamp[3] = lc_gtimer();
    // leaf lengths by symbol-order position
    int local_max = 0;
    unsigned long long local_bits = 0;
    for (int i = tid; i < k; i += LC_CB_THREADS) {
        const int d = D[parent[i]] + 1;
        const unsigned long long key = keys[i];
        lenp[(uint32_t)(key & 0xffffffffu)] = (uint8_t)(d > 255 ? 255 : d);
        local_max = max(local_max, d);
        local_bits += (key >> 32) * (unsigned long long)d;
    }
    for (int o = 16; o; o >>= 1) {
        local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
        local_bits += __shfl_xor_sync(0xffffffffu, local_bits, o);
    }
    if (lane == 0) { s_wmax[wid] = local_max; s_bits[wid] = local_bits; }
    for (int i = tid; i < NWARP * 65; i += LC_CB_THREADS) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
    // 5. canonical codes (huffman.py:58-72): within a length, consecutive
    //    codes in symbol order.  Warp w owns positions [w*span, (w+1)*span).
    const int span = (k + NWARP - 1) / NWARP;
    const int pb = min(k, wid * span), pe = min(k, pb + span);
    for (int p0 = pb; p0 < pe; p0 += 32) {
        const int pp = p0 + lane;
        const int l = pp < pe ? lenp[pp] : 0;
        if (l > 0 && l <= 64) atomicAdd(&s_wcnt[wid][l], 1);
    }
    __syncthreads();
    if (tid == 0) {
        int mx = 0;
        unsigned long long tb = 0;
        for (int w = 0; w < NWARP; ++w) { mx = max(mx, s_wmax[w]); tb += s_bits[w]; }
        out->max_len = mx;
        out->used = k;
        out->total_bits = tb;
        out->n_esc = hist[0];
        out->status = mx > 64 ? 13 : 0;
        s_wmax[0] = mx;
    }
    if (tid >= 1 && tid <= 64) {
        int acc = 0;
        for (int w = 0; w < NWARP; ++w) {
            const int c0 = s_wcnt[w][tid];
            s_wcnt[w][tid] = acc;                   // rank base of warp w within length tid
            acc += c0;
        }
        s_len_count[tid] = acc;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long code = 0;
        int prev = 0;
        for (int l = 1; l <= 64; ++l) {
            if (!s_len_count[l]) continue;
            code = (l - prev) >= 64 ? 0 : (code << (l - prev));
            s_first[l] = code;
            code += (unsigned long long)s_len_count[l];
            prev = l;
        }
        out->stamp[4] = lc_gtimer();
    }
    __syncthreads();
    if (s_wmax[0] > 64) return;
    for (int p0 = pb; p0 < pe; p0 += 32) {
        const int pp = p0 + lane;
        const int l = pp < pe ? lenp[pp] : 0;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        if (l > 0) {
            const uint32_t sy = syms[pp];
            lengths[sy] = (uint8_t)l;
            codes[sy] = s_first[l] + (unsigned long long)(s_wcnt[wid][l] + __popc(peers & ((1u << lane) - 1u)));
        }
        __syncwarp();
        if (l > 0 && (int)(__ffs(peers) - 1) == lane) s_wcnt[wid][l] += __popc(peers);
        __syncwarp();
    }
    if (tid == 0) out->stamp[5] = lc_gtimer();
}

__global__ void __launch_bounds__(LC_CB_THREADS) lc_codebook_kernel(
    const uint32_t *__restrict__ hist, uint32_t nbins, uint8_t *__restrict__ lengths,
    unsigned long long *__restrict__ codes, unsigned long long *__restrict__ gkeys,
    unsigned long long *__restrict__ ifreq_g, int *__restrict__ parent_g, LcCodebookOut *out, const LcQuantDyn *dyn,
    const unsigned long long *pending, const unsigned *maxcode)
{
    // nothing was quantized (lc_compress_auto_f64), or a chunk prediction failed and the
    // quantizer will be resumed first (the codebook and the encoder are launched again then)
    if ((dyn && dyn->skip) || (pending && *pending != ~0ULL)) {
        if (threadIdx.x == 0) { out->total_bits = 0; out->n_esc = 0; out->max_len = 0; out->used = 0; out->status = 0; }
        return;
    }
    __shared__ int s_wcnt[LC_CB_THREADS / 32][65], s_len_count[66], s_len_start[66], s_wmax[32];
    __shared__ unsigned long long s_first[66], s_bits[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < 66) s_len_count[tid] = 0;
    // 1a. used symbols per warp range (coalesced), zero all lengths.  The quantizer reports the
    // largest code it produced, so only [0, maxcode] is searched (3 symbols at eb 1e-3 instead
    // of 65,536 bins: ~20 us of this single-CTA kernel).
    const uint32_t nscan = maxcode ? min(nbins, __ldg(maxcode) + 1u) : nbins;
    const uint32_t span = ((nscan + LC_CB_THREADS / 32 - 1) / (LC_CB_THREADS / 32) + 31) & ~31u;
    const uint32_t wsb = min(nscan, wid * span), wse = min(nscan, wsb + span);
    int cnt = 0;
    for (uint32_t s0 = wsb; s0 < wse; s0 += 256) {             // 8 independent loads per lane
        uint32_t hv[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t sy = s0 + 32 * g + lane;
            hv[g] = sy < wse ? __ldg(hist + sy) : 0u;
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) cnt += __popc(__ballot_sync(0xffffffffu, hv[g] != 0));
    }
    if ((reinterpret_cast<uintptr_t>(lengths) & 15) == 0) {     // 16-byte stores
        uint4 *l4 = reinterpret_cast<uint4 *>(lengths);
        for (uint32_t i = tid; i < nbins / 16; i += LC_CB_THREADS) l4[i] = make_uint4(0, 0, 0, 0);
        for (uint32_t sy = (nbins & ~15u) + tid; sy < nbins; sy += LC_CB_THREADS) lengths[sy] = 0;
    } else {
        for (uint32_t sy = tid; sy < nbins; sy += LC_CB_THREADS) lengths[sy] = 0;
    }
    if (lane == 0) s_wcnt[wid][0] = cnt;
    __syncthreads();
    int wbase = 0, k = 0;
    for (int w = 0; w < LC_CB_THREADS / 32; ++w) {
        const int c = s_wcnt[w][0];
        if (w < wid) wbase += c;
        k += c;
    }
    __syncthreads();
    if (k == 0) {
        if (tid == 0) { out->total_bits = 0; out->n_esc = 0; out->max_len = 0; out->used = 0; out->status = 0; }
        return;
    }
    if (k <= LC_CB_SMEM_KEYS)
        lc_codebook_body<true>(hist, nbins, lengths, codes, gkeys, ifreq_g, parent_g, out, k, wbase, wsb, wse,
                               s_len_count, s_len_start, s_first, s_bits, s_wmax, s_wcnt);
    else
        lc_codebook_body<false>(hist, nbins, lengths, codes, gkeys, ifreq_g, parent_g, out, k, wbase, wsb, wse,
                                s_len_count, s_len_start, s_first, s_bits, s_wmax, s_wcnt);
}

// ---------------------------------------------------------------------------
// encoder



__global__ void lc_zero_words_kernel(uint32_t *__restrict__ p, const LcCodebookOut *__restrict__ cb)
{
    const uint64_t nw = (cb->total_bits + 31) >> 5;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += stride) p[i] = 0;
}

__device__ __forceinline__ void lc_put_word(uint32_t *payload, uint64_t w, uint32_t bits_be, bool shared)
{
    const uint32_t le = __byte_perm(bits_be, 0, 0x0123);   // MSB-first bytes
    if (shared) atomicOr(payload + w, le);
    else payload[w] = le;
}

// Encoder.  A tile of LC_TILE symbols per CTA iteration, 32 consecutive
// symbols per thread held in registers.  Tile bit offsets come from a
// decoupled look-back over (bits, escapes) run by warp 0 while the other warps
// assemble the tile's bit string at bit alignment 0 in a shared-memory word
// buffer (thread-boundary words merged with shared atomics); the string is
// written out shifted by (tile offset % 32) with coalesced word stores, merging
// only the tile's first and last words with the neighbouring tiles (the
// payload is zeroed first).  huffman.encode (huffman.py:52-72) packs MSB-first.
#define LC_ENC_WBUF 4096                 // tile buffer words (16 bits per symbol on average)
#define LC_ENC_NT (LC_TPB + 32)          // 8 packing warps + 1 look-back warp

template <typename CodeT>
struct LcCodeRegs {
    static constexpr int NW = LC_L * sizeof(CodeT) / 4;   // 32-bit words holding 32 symbols
    uint32_t w[NW];
    __device__ __forceinline__ uint32_t get(int j) const
    {
        if (sizeof(CodeT) == 2) return (w[j >> 1] >> (16 * (j & 1))) & 0xffffu;
        return w[j];
    }
};

template <typename CodeT>
__global__ void __launch_bounds__(LC_ENC_NT, 4) lc_encode_kernel(LcEncParams P)
{
    if (P.dyn && P.dyn->skip) return;
    if (P.pending && *P.pending != ~0ULL) return;    // the quantizer is resumed first
    typedef cub::BlockScan<unsigned long long, LC_ENC_NT> ScanU;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    uint32_t *tpk = reinterpret_cast<uint32_t *>(lc_dyn_smem);   // (len << 27) | code
    uint32_t *wbuf = tpk + LC_ENC_TAB;
    __shared__ typename ScanU::TempStorage scan_tmp;
    __shared__ long long sh_tile;
    __shared__ unsigned long long sh_in_bits, sh_in_esc;
    const int tid = threadIdx.x;
    const CodeT *codes = reinterpret_cast<const CodeT *>(P.codes);
    const bool fast = P.cb->max_len <= 32;
    const bool packed = P.cb->max_len <= 27;              // codes fit the 32-bit table entries
    const uint32_t tab = packed ? (P.nbins < LC_ENC_TAB ? P.nbins : LC_ENC_TAB) : 0u;
    for (uint32_t s = tid; s < tab; s += LC_ENC_NT)
        tpk[s] = ((uint32_t)P.lengths[s] << 27) | (uint32_t)P.cw[s];
    auto unpack = [](uint32_t t) -> unsigned long long {
        return ((unsigned long long)(t >> 27) << 32) | (t & 0x7ffffffu);
    };
    auto entry = [&](uint32_t s) -> unsigned long long {
        return s < tab ? unpack(tpk[s]) : (((unsigned long long)P.lengths[s] << 32) | (uint32_t)P.cw[s]);
    };

    for (;;) {
        __syncthreads();
        if (tid == 0) sh_tile = atomicAdd(P.tile_counter, 1u);
        __syncthreads();
        const long long t = sh_tile;
        if (t >= (long long)P.ntiles) break;
        const long long p0 = t * (long long)LC_TILE + (long long)tid * LC_L;
        // warps 0..7 pack 32 symbols per thread; warp 8 only runs the look-back
        const int len = tid < LC_TPB ? (int)max(0LL, min((long long)LC_L, (long long)P.m - p0)) : 0;
        LcCodeRegs<CodeT> C;
        if (len == LC_L) {
            const uint4 *src = reinterpret_cast<const uint4 *>(codes + p0);
#pragma unroll
            for (int k = 0; k < LcCodeRegs<CodeT>::NW / 4; ++k) {
                const uint4 v = __ldcs(src + k);
                C.w[4 * k] = v.x; C.w[4 * k + 1] = v.y; C.w[4 * k + 2] = v.z; C.w[4 * k + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < LcCodeRegs<CodeT>::NW; ++k) C.w[k] = 0;
#pragma unroll
            for (int j = 0; j < LC_L; ++j) {
                if (j < len) {
                    const uint32_t v = (uint32_t)codes[p0 + j];
                    if (sizeof(CodeT) == 2) C.w[j >> 1] |= v << (16 * (j & 1));
                    else C.w[j] = v;
                }
            }
        }
        // full chunk with every symbol in the smem table: no per-symbol guards
        uint32_t cmax = 0;
#pragma unroll
        for (int k = 0; k < LcCodeRegs<CodeT>::NW; ++k) cmax = sizeof(CodeT) == 2 ? __vmaxu2(cmax, C.w[k]) : max(cmax, C.w[k]);
        if (sizeof(CodeT) == 2) cmax = max(cmax & 0xffffu, cmax >> 16);
        const bool tabled = len == LC_L && cmax < tab;
        uint32_t bits32 = 0, nesc32 = 0;
        if (tabled) {
#pragma unroll
            for (int j = 0; j < LC_L; ++j) bits32 += tpk[C.get(j)] >> 27;
#pragma unroll
            for (int k = 0; k < LcCodeRegs<CodeT>::NW; ++k)
                nesc32 += sizeof(CodeT) == 2 ? __popc(__vcmpeq2(C.w[k], 0u)) >> 4 : (C.w[k] == 0u);
        } else {
#pragma unroll
            for (int j = 0; j < LC_L; ++j) {
                if (j < len) {
                    const uint32_t s = C.get(j);
                    bits32 += (uint32_t)(entry(s) >> 32);
                    nesc32 += (s == 0);
                }
            }
        }
        const unsigned long long bits = bits32, nesc = nesc32;
        // per-tile bits < 2^20 and escapes < 2^14: one scan of (esc << 32 | bits)
        unsigned long long ex, agg;
        ScanU(scan_tmp).ExclusiveSum(bits | (nesc << 32), ex, agg);
        const unsigned long long abits = agg & 0xffffffffull, aesc = agg >> 32;
        const unsigned nwt0 = (unsigned)((abits + 31) >> 5);       // tile words at bit alignment 0
        const bool fast_tile = fast && nwt0 + 1 <= LC_ENC_WBUF;
        LcEncDesc *d = P.desc + t;
        if (tid == 0 && t > 0) {                                     // publish the aggregate first
            __stcg(&d->agg_bits, abits);
            __stcg(&d->agg_esc, aesc);
            st_release(&d->st, 1);
        }
        // Tile offsets by a decoupled look-back run by warp 0 while the other warps
        // pack the tile's bits at alignment 0 (the shift by B0 % 32 happens on the
        // way out), so the look-back latency overlaps the packing.
        auto lookback = [&]() {
            ulonglong2 in = make_ulonglong2(0, 0);
            if (t > 0)
                in = lc_lookback_warp<ulonglong2>(
                    t, make_ulonglong2(0, 0),
                    [](const ulonglong2 &a, const ulonglong2 &b) { return make_ulonglong2(a.x + b.x, a.y + b.y); },
                    [](const ulonglong2 &v, int o) {
                        return make_ulonglong2(__shfl_down_sync(0xffffffffu, v.x, o),
                                               __shfl_down_sync(0xffffffffu, v.y, o));
                    },
                    [&](long long k) { return ld_acquire(&P.desc[k].st); },
                    [&](long long k, int st) {
                        return st == 2 ? make_ulonglong2(__ldcg(&P.desc[k].incl_bits), __ldcg(&P.desc[k].incl_esc))
                                       : make_ulonglong2(__ldcg(&P.desc[k].agg_bits), __ldcg(&P.desc[k].agg_esc));
                    });
            if (tid == LC_TPB) {
                __stcg(&d->incl_bits, in.x + abits);
                __stcg(&d->incl_esc, in.y + aesc);
                st_release(&d->st, 2);
                sh_in_bits = in.x; sh_in_esc = in.y;
            }
        };
        if (fast_tile) {
            for (unsigned i = tid; i <= nwt0; i += LC_ENC_NT) wbuf[i] = 0;
            __syncthreads();
            if (tid >= LC_TPB) lookback();
            if (bits) {
                const unsigned lb = (unsigned)(ex & 0xffffffffull);            // bit in the tile buffer
                const unsigned wfirst = lb >> 5, wlast = (unsigned)((lb + bits - 1) >> 5);
                unsigned w = wfirst;
                unsigned long long acc = 0;
                int nb = (int)(lb & 31);
                auto put = [&](unsigned long long e) {
                    const int l = (int)(e >> 32);
                    acc = (acc << l) | (uint32_t)e;
                    nb += l;
                    if (nb >= 32) {
                        nb -= 32;
                        const uint32_t word = (uint32_t)(acc >> nb);
                        if (w == wfirst || w == wlast) atomicOr(wbuf + w, word);
                        else wbuf[w] = word;
                        ++w;
                    }
                };
                if (tabled) {
#pragma unroll
                    for (int j = 0; j < LC_L; ++j) put(unpack(tpk[C.get(j)]));
                } else {
#pragma unroll
                    for (int j = 0; j < LC_L; ++j)
                        if (j < len) put(entry(C.get(j)));
                }
                if (nb > 0) atomicOr(wbuf + w, (uint32_t)(acc << (32 - nb)));
            }
            __syncthreads();
        } else {
            if (tid >= LC_TPB) lookback();
            __syncthreads();
        }
        const unsigned long long B0 = sh_in_bits;
        // v2 sync table: bit offset of every LC_SYNC_K-th symbol
        if (P.sync && len > 0 && (p0 & (LC_SYNC_K - 1)) == 0) {
            P.sync[p0 / LC_SYNC_K] = B0 + (ex & 0xffffffffull);
            if (P.sync_esc) P.sync_esc[p0 / LC_SYNC_K] = sh_in_esc + (ex >> 32);
        }
        // escapes (compressor.py:409-410): code index i-1 <-> element i
        if (nesc) {
            unsigned long long e = sh_in_esc + (ex >> 32);
#pragma unroll
            for (int j = 0; j < LC_L; ++j)
                if (j < len && C.get(j) == 0) {
                    const unsigned long long el = (unsigned long long)(p0 + j + 1);
                    if (e < P.esc_cap) {
                        P.esc_idx[e] = el;
                        P.esc_val[e] = P.x ? P.x[el] : 0.0;
                    }
                    ++e;
                }
        }
        if (fast_tile) {
            // out word i of the tile = the alignment-0 stream shifted right by s = B0 % 32
            const unsigned sft = (unsigned)(B0 & 31);
            const unsigned nout = (unsigned)((sft + abits + 31) >> 5);
            const unsigned long long gw0 = B0 >> 5;
            for (unsigned i = tid; i < nout; i += LC_ENC_NT) {
                const uint32_t cur = i < nwt0 ? wbuf[i] : 0u;
                const uint32_t prev = (i > 0 && sft) ? wbuf[i - 1] : 0u;
                const uint32_t word = sft ? ((cur >> sft) | (prev << (32 - sft))) : cur;
                const uint32_t v = __byte_perm(word, 0, 0x0123);       // MSB-first bytes
                if (i == 0 || i + 1 == nout) atomicOr(P.payload + gw0 + i, v);
                else P.payload[gw0 + i] = v;
            }
        } else if (bits) {
            // long codes or a very long tile: pack straight into global words
            const unsigned long long b0 = B0 + (ex & 0xffffffffull);
            const unsigned long long b1 = b0 + bits;
            const uint64_t w0 = b0 >> 5, wl = (b1 - 1) >> 5;
            uint64_t w = w0;
            uint64_t buf = 0;
            int nb = (int)(b0 & 31);
            for (int j = 0; j < len; ++j) {
                const uint32_t s = (uint32_t)codes[p0 + j];
                int l = P.lengths[s];
                const unsigned long long cw = P.cw[s];
                while (l > 0) {
                    const int take = l > 32 ? l - 32 : l;      // high part first
                    const uint64_t piece = (cw >> (l - take)) & ((take == 64) ? ~0ULL : ((1ULL << take) - 1));
                    buf = (buf << take) | piece;
                    nb += take;
                    l -= take;
                    if (nb >= 32) {
                        const uint32_t word = (uint32_t)(buf >> (nb - 32));
                        lc_put_word(P.payload, w, word, w == w0 || w == wl);
                        ++w;
                        nb -= 32;
                        buf &= (nb ? ((1ULL << nb) - 1) : 0ULL);
                    }
                }
            }
            if (nb > 0) lc_put_word(P.payload, w, (uint32_t)(buf << (32 - nb)), true);
        }
    }
}

size_t lc_codebook_smem_bytes()
{
    return (2 * sizeof(unsigned long long) + 2 * sizeof(int) + sizeof(uint32_t) + 1) * LC_CB_SMEM_KEYS;
}
size_t lc_encode_smem_bytes()
{
    return sizeof(uint32_t) * LC_ENC_TAB + sizeof(uint32_t) * LC_ENC_WBUF;
}

template __global__ void lc_encode_kernel<uint16_t>(LcEncParams);
template __global__ void lc_encode_kernel<uint32_t>(LcEncParams);
