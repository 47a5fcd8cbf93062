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
#include <cub/block/block_scan.cuh>
#include "lc_kernels.cuh"

#define LC_CB_THREADS 1024
#define LC_CB_SMEM_KEYS 8192
#define LC_ENC_TAB 4096


__device__ void lc_bitonic_sort(unsigned long long *a, int npow2)
{
    for (int k = 2; k <= npow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long ai = a[i], aj = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((ai > aj) == up) { a[i] = aj; a[ixj] = ai; }
                }
            }
            __syncthreads();
        }
    }
}

// hist[nbins] -> lengths[nbins], codes[nbins], meta.  scratch holds
// 3*nbins u64 + 2*nbins int32 (global fallback storage).
__global__ void __launch_bounds__(LC_CB_THREADS) lc_codebook_kernel(
    const uint32_t *__restrict__ hist, uint32_t nbins, uint8_t *__restrict__ lengths,
    unsigned long long *__restrict__ codes, unsigned long long *__restrict__ gkeys,
    unsigned long long *__restrict__ ifreq, int *__restrict__ parent, LcCodebookOut *out)
{
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    unsigned long long *skeys = reinterpret_cast<unsigned long long *>(lc_dyn_smem);
    __shared__ int s_used, s_len_count[66];
    __shared__ unsigned long long s_first[66];
    __shared__ unsigned long long s_bits[32];
    const int tid = threadIdx.x;
    if (tid == 0) s_used = 0;
    if (tid < 66) s_len_count[tid] = 0;
    __syncthreads();

    // 1. used symbols (order irrelevant: sorted next)
    int cnt = 0;
    for (uint32_t s = tid; s < nbins; s += blockDim.x) cnt += hist[s] > 0;
    const int base = atomicAdd(&s_used, cnt) ; (void)base;
    __syncthreads();
    const int k = s_used;
    int npow2 = 1;
    while (npow2 < k) npow2 <<= 1;
    unsigned long long *keys = (npow2 <= LC_CB_SMEM_KEYS) ? skeys : gkeys;
    __syncthreads();
    if (tid == 0) s_used = 0;
    __syncthreads();
    for (uint32_t s = tid; s < nbins; s += blockDim.x) {
        lengths[s] = 0;
        codes[s] = 0;
        if (hist[s]) {
            const int pos = atomicAdd(&s_used, 1);
            keys[pos] = ((unsigned long long)hist[s] << 32) | s;
        }
    }
    __syncthreads();
    for (int i = k + tid; i < npow2; i += blockDim.x) keys[i] = ~0ULL;
    __syncthreads();
    if (k == 0) {
        if (tid == 0) { out->total_bits = 0; out->n_esc = 0; out->max_len = 0; out->used = 0; out->status = 0; }
        return;
    }
    if (k == 1) {                                   // huffman.py:33-35
        if (tid == 0) {
            const uint32_t s = (uint32_t)(keys[0] & 0xffffffffu);
            lengths[s] = 1;
            codes[s] = 0;
            out->total_bits = keys[0] >> 32;
            out->n_esc = hist[0];
            out->max_len = 1; out->used = 1; out->status = 0;
        }
        return;
    }
    // 2. sort by (freq, symbol)
    lc_bitonic_sort(keys, npow2);

    // 3. two-queue merge (thread 0).  Leaves 0..k-1 in sorted order; internal
    //    node m (0..k-2) has freq ifreq[m]; parent[] indexes internal nodes:
    //    parent[leaf] at [0,k), parent[k + m] for internal node m.
    if (tid == 0) {
        int li = 0, ii = 0;                          // queue heads
        for (int m = 0; m < k - 1; ++m) {
            int pick[2];
            unsigned long long f[2];
            for (int q = 0; q < 2; ++q) {
                const bool leaf_ok = li < k;
                const bool int_ok = ii < m;
                const unsigned long long lf = leaf_ok ? (keys[li] >> 32) : ~0ULL;
                const unsigned long long nf = int_ok ? ifreq[ii] : ~0ULL;
                if (leaf_ok && (!int_ok || lf <= nf)) { pick[q] = li; f[q] = lf; ++li; }
                else { pick[q] = k + ii; f[q] = nf; ++ii; }
            }
            ifreq[m] = f[0] + f[1];
            parent[pick[0]] = m;
            parent[pick[1]] = m;
        }
    }
    __syncthreads();
    // 4. depths: internal nodes in reverse creation order (root = k-2)
    int *depth = reinterpret_cast<int *>(ifreq);     // reuse (freqs no longer needed)
    if (tid == 0) {
        depth[k - 2] = 0;
        for (int m = k - 3; m >= 0; --m) depth[m] = depth[parent[k + m]] + 1;
    }
    __syncthreads();
    int local_max = 0;
    unsigned long long local_bits = 0;
    for (int i = tid; i < k; i += blockDim.x) {
        const int d = depth[parent[i]] + 1;
        const uint32_t s = (uint32_t)(keys[i] & 0xffffffffu);
        lengths[s] = (uint8_t)(d > 255 ? 255 : d);
        if (d <= 64) atomicAdd(&s_len_count[d], 1);
        local_max = max(local_max, d);
        local_bits += (keys[i] >> 32) * (unsigned long long)d;
    }
    for (int o = 16; o; o >>= 1) {
        local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
        local_bits += __shfl_xor_sync(0xffffffffu, local_bits, o);
    }
    __shared__ int s_wmax[32];
    if ((tid & 31) == 0) { s_wmax[tid >> 5] = local_max; s_bits[tid >> 5] = local_bits; }
    __syncthreads();
    if (tid == 0) {
        int mx = 0;
        unsigned long long tb = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { mx = max(mx, s_wmax[w]); tb += s_bits[w]; }
        out->max_len = mx;
        out->used = k;
        out->total_bits = tb;
        out->n_esc = hist[0];
        out->status = mx > 64 ? 13 : 0;
        // canonical first codes per length (huffman.py:64-71)
        unsigned long long code = 0;
        int prev = 0;
        for (int l = 1; l <= 64; ++l) {
            if (!s_len_count[l]) continue;
            code = (l - prev) >= 64 ? 0 : (code << (l - prev));
            s_first[l] = code;
            code += (unsigned long long)s_len_count[l];
            // last code of this length is code-1; the next length shifts it
            prev = l;
        }
    }
    __syncthreads();
    if (out->status) return;
    // 5. codes: symbols of one length get consecutive codes in symbol order.
    //    Warp w owns a contiguous symbol range: count lengths, scan the counts
    //    across warps, then assign ranks with match_any inside each group.
    __shared__ int s_wcnt[LC_CB_THREADS / 32][65];
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    for (int i = tid; i < nw * 65; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t span = (nbins + nw - 1) / nw;
    const uint32_t sb = wid * span, se = min(nbins, sb + span);
    for (uint32_t s0 = sb; s0 < se; s0 += 32) {
        const uint32_t s = s0 + lane;
        const int l = s < se ? lengths[s] : 0;
        if (l > 0) atomicAdd(&s_wcnt[wid][l], 1);
    }
    __syncthreads();
    if (tid >= 1 && tid <= 64 && s_len_count[tid]) {
        unsigned long long off = s_first[tid];
        for (int w = 0; w < nw; ++w) {
            const int c0 = s_wcnt[w][tid];
            s_wcnt[w][tid] = (int)(off - s_first[tid]);   // exclusive rank base
            off += c0;
        }
    }
    __syncthreads();
    for (uint32_t s0 = sb; s0 < se; s0 += 32) {
        const uint32_t s = s0 + lane;
        const int l = s < se ? lengths[s] : 0;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        if (l > 0) {
            const int rank = __popc(peers & ((1u << lane) - 1u));
            codes[s] = s_first[l] + (unsigned long long)(s_wcnt[wid][l] + rank);
        }
        __syncwarp();
        if (l > 0 && (int)(__ffs(peers) - 1) == lane) s_wcnt[wid][l] += __popc(peers);
        __syncwarp();
    }
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

template <typename CodeT>
__global__ void __launch_bounds__(LC_TPB) lc_encode_kernel(LcEncParams P)
{
    typedef cub::BlockScan<unsigned long long, LC_TPB> ScanU;
    extern __shared__ __align__(16) unsigned char lc_dyn_smem[];
    unsigned long long *tcw = reinterpret_cast<unsigned long long *>(lc_dyn_smem);
    uint32_t *cs = reinterpret_cast<uint32_t *>(tcw + LC_ENC_TAB);
    uint8_t *tlen = reinterpret_cast<uint8_t *>(cs + LC_TPB * LC_ROW);
    __shared__ typename ScanU::TempStorage scan_tmp;
    __shared__ long long sh_tile;
    __shared__ unsigned long long sh_in_bits, sh_in_esc;
    __shared__ ulonglong2 lb_u2[LC_TPB / 32], lb_u2_res;
    __shared__ int sh_j;
    const int tid = threadIdx.x;
    const CodeT *codes = reinterpret_cast<const CodeT *>(P.codes);
    const uint32_t tab = P.nbins < LC_ENC_TAB ? P.nbins : LC_ENC_TAB;
    for (uint32_t s = tid; s < tab; s += LC_TPB) { tlen[s] = P.lengths[s]; tcw[s] = P.cw[s]; }

    for (;;) {
        __syncthreads();
        if (tid == 0) sh_tile = atomicAdd(P.tile_counter, 1u);
        __syncthreads();
        const long long t = sh_tile;
        if (t >= (long long)P.ntiles) break;
        const long long base = t * (long long)LC_TILE;
#pragma unroll 8
        for (int k = 0; k < LC_L; ++k) {
            const int off = k * LC_TPB + tid;
            const long long pos = base + off;
            cs[(off >> 5) * LC_ROW + (off & 31)] = pos < (long long)P.m ? (uint32_t)codes[pos] : 0xffffffffu;
        }
        __syncthreads();
        const uint32_t *row = cs + tid * LC_ROW;
        const long long p0 = base + (long long)tid * LC_L;
        const int len = (int)max(0LL, min((long long)LC_L, (long long)P.m - p0));
        unsigned long long bits = 0, nesc = 0;
        for (int j = 0; j < len; ++j) {
            const uint32_t s = row[j];
            bits += s < LC_ENC_TAB ? tlen[s] : P.lengths[s];
            nesc += (s == 0);
        }
        unsigned long long bex, eex, bagg, eagg;
        ScanU(scan_tmp).ExclusiveSum(bits, bex, bagg);
        __syncthreads();
        ScanU(scan_tmp).ExclusiveSum(nesc, eex, eagg);
        {
            LcEncDesc *d = P.desc + t;
            ulonglong2 in = make_ulonglong2(0, 0);
            if (t > 0) {
                if (tid == 0) {
                    __stcg(&d->agg_bits, bagg);
                    __stcg(&d->agg_esc, eagg);
                    st_release(&d->st, 1);
                }
                in = lc_lookback_block<ulonglong2>(
                    t, make_ulonglong2(0, 0),
                    [](const ulonglong2 &a, const ulonglong2 &b) { return make_ulonglong2(a.x + b.x, a.y + b.y); },
                    [](const ulonglong2 &v, int o) {
                        return make_ulonglong2(__shfl_down_sync(0xffffffffu, v.x, o),
                                               __shfl_down_sync(0xffffffffu, v.y, o));
                    },
                    [&](long long k) { return &P.desc[k].st; },
                    [&](long long k, int st) {
                        return st == 2 ? make_ulonglong2(__ldcg(&P.desc[k].incl_bits), __ldcg(&P.desc[k].incl_esc))
                                       : make_ulonglong2(__ldcg(&P.desc[k].agg_bits), __ldcg(&P.desc[k].agg_esc));
                    },
                    lb_u2, &sh_j, &lb_u2_res);
            }
            if (tid == 0) {
                __stcg(&d->incl_bits, in.x + bagg);
                __stcg(&d->incl_esc, in.y + eagg);
                st_release(&d->st, 2);
                sh_in_bits = in.x; sh_in_esc = in.y;
            }
        }
        __syncthreads();
        // escapes (compressor.py:409-410): code index i-1 <-> element i
        if (nesc) {
            unsigned long long e = sh_in_esc + eex;
            for (int j = 0; j < len; ++j)
                if (row[j] == 0) {
                    const unsigned long long el = (unsigned long long)(p0 + j + 1);
                    P.esc_idx[e] = el;
                    P.esc_val[e] = P.x ? P.x[el] : 0.0;
                    ++e;
                }
        }
        if (len == 0) continue;
        // bit packing
        const unsigned long long b0 = sh_in_bits + bex;
        const unsigned long long b1 = b0 + bits;
        const uint64_t w0 = b0 >> 5, wl = (b1 - 1) >> 5;
        uint64_t w = w0;
        uint64_t buf = 0;
        int nb = (int)(b0 & 31);                   // leading zero bits of the first word
        for (int j = 0; j < len; ++j) {
            const uint32_t s = row[j];
            int l = s < LC_ENC_TAB ? tlen[s] : P.lengths[s];
            const unsigned long long cw = s < LC_ENC_TAB ? tcw[s] : P.cw[s];
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
        if (nb > 0) {
            const uint32_t word = (uint32_t)(buf << (32 - nb));
            lc_put_word(P.payload, w, word, true);
        }
    }
}

size_t lc_codebook_smem_bytes() { return sizeof(unsigned long long) * LC_CB_SMEM_KEYS; }
size_t lc_encode_smem_bytes()
{
    return sizeof(unsigned long long) * LC_ENC_TAB + sizeof(uint32_t) * LC_TPB * LC_ROW + LC_ENC_TAB;
}

template __global__ void lc_encode_kernel<uint16_t>(LcEncParams);
template __global__ void lc_encode_kernel<uint32_t>(LcEncParams);
