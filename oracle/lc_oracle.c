/*
 * lc_oracle.c -- CPU restatement of the reference lossy-checkpoint compressor.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_1805_07384_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product path never calls it (there is no CPU fallback).
 *
 * Every function restates one reference routine (Python + numba, under
 * /root/reference/pkg/src/lossyckpt) with the same IEEE-754 binary64
 * semantics: plain mul/add/div, no FMA contraction (build with
 * -ffp-contract=off; SSE2 scalar doubles), floor() for np.floor.
 *
 * Parity is pinned against golden vectors produced by running the real
 * reference (tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LCO_ESCAPE_CODE 0

/* compressor.py:319-355  _compress_kernel.
 * Closed-loop order-1 predictor + uniform quantizer with bin width 2*eb_abs.
 * Returns the escape count; esc_idx receives the escaped positions.       */
int64_t lco_compress_kernel(const double *data, int64_t n, double eb_abs,
                            int64_t n_bins_half, int record, int64_t *codes,
                            double *recon, double *pe_out, double *pe_rec_out,
                            int64_t *esc_idx_buf)
{
    const double delta = 2.0 * eb_abs;              /* compressor.py:323 */
    double prev = data[0];                          /* :324 */
    int64_t n_esc = 0;
    const double max_m = (double)(n_bins_half - 1); /* :327 */
    if (recon) recon[0] = prev;
    for (int64_t i = 1; i < n; ++i) {               /* :328 */
        const double v = data[i];
        const double pred = prev;
        const double pe = v - pred;                 /* :331 */
        const double q = pe / delta + 0.5;          /* :332 */
        int escape = 1;
        int64_t m = 0;
        double cand = prev;
        if (q >= -max_m && q < max_m + 1.0) {       /* :336 */
            m = (int64_t)floor(q);                  /* :337 */
            cand = (m == 0) ? pred : pred + (double)m * delta; /* :338 */
            if (fabs(v - cand) <= eb_abs) escape = 0; /* :340 */
        }
        if (escape) {                               /* :342-346 */
            codes[i - 1] = LCO_ESCAPE_CODE;
            esc_idx_buf[n_esc++] = i;
            prev = v;
        } else {                                    /* :347-350 */
            const int64_t zz = m >= 0 ? 2 * m : -2 * m - 1;
            codes[i - 1] = zz + 1;
            prev = cand;
        }
        if (recon) recon[i] = prev;                 /* :351 */
        if (record) {                               /* :352-354 */
            pe_out[i - 1] = pe;
            pe_rec_out[i - 1] = prev - pred;
        }
    }
    return n_esc;
}

/* compressor.py:358-376  _decompress_kernel.  Returns escapes consumed, or
 * -1 when the codes need more escape values than supplied.                */
int64_t lco_decompress_kernel(const int64_t *codes, int64_t n, double first_value,
                              double delta, const double *escape_values,
                              int64_t n_esc_values, double *out)
{
    double prev = first_value;
    out[0] = prev;
    int64_t e = 0;
    for (int64_t i = 1; i < n; ++i) {
        const int64_t c = codes[i - 1];
        if (c == LCO_ESCAPE_CODE) {
            if (e >= n_esc_values) return -1;
            prev = escape_values[e++];
        } else {
            const int64_t zz = c - 1;
            const int64_t m = (zz >> 1) ^ -(zz & 1);
            if (m != 0) prev = prev + (double)m * delta;
        }
        out[i] = prev;
    }
    return e;
}

/* ---------------------------------------------------------------------- */
/* huffman.py:21-55  code_lengths: heapq Huffman with (freq, counter) keys. */

typedef struct { int64_t freq; int64_t counter; int64_t node; } lco_hent;

static int hless(const lco_hent *a, const lco_hent *b)
{
    return a->freq < b->freq || (a->freq == b->freq && a->counter < b->counter);
}

static void hsift_down(lco_hent *h, int64_t n, int64_t i)
{
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, s = i;
        if (l < n && hless(&h[l], &h[s])) s = l;
        if (r < n && hless(&h[r], &h[s])) s = r;
        if (s == i) return;
        lco_hent t = h[i]; h[i] = h[s]; h[s] = t; i = s;
    }
}

static void hsift_up(lco_hent *h, int64_t i)
{
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!hless(&h[i], &h[p])) return;
        lco_hent t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}

/* Returns 0 on success, -1 on a negative frequency (ParameterError). */
int lco_code_lengths(const int64_t *freqs, int64_t k, uint8_t *lengths)
{
    int64_t used = 0, last = -1;
    for (int64_t s = 0; s < k; ++s) {
        if (freqs[s] < 0) return -1;               /* huffman.py:27-28 */
        lengths[s] = 0;
        if (freqs[s] > 0) { ++used; last = s; }
    }
    if (used == 0) return 0;                        /* :31-32 */
    if (used == 1) { lengths[last] = 1; return 0; } /* :33-35 */
    /* nodes 0..used-1 are leaves (symbol order), used.. are internal      */
    int64_t cap = 2 * used;
    lco_hent *heap = (lco_hent *)malloc(sizeof(lco_hent) * used);
    int64_t *sym = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t *left = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t *right = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t *depth = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t nn = 0, counter = 0;
    for (int64_t s = 0; s < k; ++s) {               /* :36-40 */
        if (freqs[s] > 0) {
            sym[nn] = s; left[nn] = right[nn] = -1;
            heap[nn].freq = freqs[s]; heap[nn].counter = counter++; heap[nn].node = nn;
            ++nn;
        }
    }
    int64_t hn = nn;
    for (int64_t i = hn / 2 - 1; i >= 0; --i) hsift_down(heap, hn, i); /* heapify */
    while (hn > 1) {                                /* :42-46 */
        lco_hent a = heap[0]; heap[0] = heap[--hn]; hsift_down(heap, hn, 0);
        lco_hent b = heap[0]; heap[0] = heap[--hn]; hsift_down(heap, hn, 0);
        left[nn] = a.node; right[nn] = b.node; sym[nn] = -1;
        heap[hn].freq = a.freq + b.freq; heap[hn].counter = counter++; heap[hn].node = nn;
        hsift_up(heap, hn); ++hn; ++nn;
    }
    /* depth-first walk from the root (:47-54); internal nodes were created in
     * increasing index order, so walking indices downward visits parents
     * before children.                                                    */
    depth[nn - 1] = 0;
    for (int64_t v = nn - 1; v >= 0; --v) {
        if (left[v] >= 0) { depth[left[v]] = depth[v] + 1; depth[right[v]] = depth[v] + 1; }
        else lengths[sym[v]] = (uint8_t)depth[v];
    }
    free(heap); free(sym); free(left); free(right); free(depth);
    return 0;
}

/* huffman.py:58-72  canonical_codes.  Returns -1 if a length exceeds 64.  */
int lco_canonical_codes(const uint8_t *lengths, int64_t k, uint64_t *codes)
{
    int64_t count[65] = {0};
    for (int64_t s = 0; s < k; ++s) {
        if (lengths[s] > 64) return -1;             /* huffman.py:61-62 */
        codes[s] = 0;
        count[lengths[s]]++;
    }
    /* walk (length, symbol) in sorted order (:64-71) */
    uint64_t code = 0;
    int prev_len = 0;
    for (int len = 1; len <= 64; ++len) {
        if (!count[len]) continue;
        for (int64_t s = 0; s < k; ++s) {
            if (lengths[s] != len) continue;
            code = (len - prev_len) >= 64 ? 0 : code << (len - prev_len);
            codes[s] = code;
            code += 1;
            prev_len = len;
        }
    }
    return 0;
}

/* huffman.py:96-107  _encode_kernel: MSB-first bit packing.  `out` must be
 * zeroed and hold ceil(total_bits/8) bytes.  Returns bits written.        */
uint64_t lco_encode_kernel(const int64_t *symbols, int64_t n, const uint64_t *codes,
                           const uint8_t *lengths, uint8_t *out)
{
    uint64_t bitpos = 0;
    for (int64_t idx = 0; idx < n; ++idx) {
        const int64_t sym = symbols[idx];
        const uint64_t code = codes[sym];
        const int length = lengths[sym];
        for (int kk = length - 1; kk >= 0; --kk) {
            if ((code >> kk) & 1u) out[bitpos >> 3] |= (uint8_t)(1u << (7 - (bitpos & 7)));
            ++bitpos;
        }
    }
    return bitpos;
}

/* huffman.py:75-93 + 110-132  _decode_tables + _decode_kernel.
 * Returns 0 ok, 1 invalid codeword, 2 payload exhausted, 3 trailing bits. */
int lco_decode_kernel(const uint8_t *payload, uint64_t bit_length, const uint8_t *lengths,
                      int64_t k, int64_t count, int64_t *out)
{
    int max_len = 0;
    for (int64_t s = 0; s < k; ++s) if (lengths[s] > max_len) max_len = lengths[s];
    int64_t counts[66] = {0}, first_code[66] = {0}, offsets[66] = {0};
    for (int64_t s = 0; s < k; ++s) if (lengths[s]) counts[lengths[s]]++;
    int64_t code = 0, offset = 0;
    for (int len = 1; len <= max_len; ++len) {       /* :86-90 */
        first_code[len] = code; offsets[len] = offset;
        code = (code + counts[len]) << 1;            /* int64 wrap like numpy */
        offset += counts[len];
    }
    int64_t *sorted = (int64_t *)malloc(sizeof(int64_t) * (offset > 0 ? offset : 1));
    {
        int64_t pos[66];
        for (int len = 1; len <= max_len; ++len) pos[len] = offsets[len];
        for (int64_t s = 0; s < k; ++s) if (lengths[s]) sorted[pos[lengths[s]]++] = s;
    }
    uint64_t bitpos = 0;
    for (int64_t idx = 0; idx < count; ++idx) {      /* :114-129 */
        int64_t c = 0; int length = 0;
        for (;;) {
            if (bitpos >= bit_length) { free(sorted); return 2; }
            const int bit = (payload[bitpos >> 3] >> (7 - (bitpos & 7))) & 1;
            ++bitpos;
            c = (c << 1) | bit;
            ++length;
            if (length > max_len) { free(sorted); return 1; }
            const int64_t rel = c - first_code[length];
            if (0 <= rel && rel < counts[length]) { out[idx] = sorted[offsets[length] + rel]; break; }
        }
    }
    free(sorted);
    return bitpos != bit_length ? 3 : 0;             /* :130-132 */
}

/* Test-input generator (not a reference routine): the adversarial bin-edge
 * corpus of SURVEY.md 8.P.  Advances the reference chain (compressor.py:
 * 329-351, same operations as lco_compress_kernel) and places every x_i at
 * prev + (m_i - 0.5) * delta moved by k_i ulps (|k_i| <= 3), i.e. within a few
 * ulps of a bin edge of the reference's own prediction.  m and k are drawn by
 * numpy (tests/stress_inputs.py) so the corpus is reproducible everywhere.  */
void lco_edge_corpus(const int64_t *m, const int64_t *k, int64_t n, double x0, double eb,
                     int64_t n_bins_half, double *out)
{
    const double delta = 2.0 * eb;
    const double max_m = (double)(n_bins_half - 1);
    double prev = x0;
    out[0] = x0;
    for (int64_t i = 1; i < n; ++i) {
        const double edge = prev + ((double)m[i - 1] - 0.5) * delta;
        double v = edge;
        const int64_t kk = k[i - 1];
        for (int64_t j = 0; j < (kk < 0 ? -kk : kk); ++j) v = nextafter(v, kk > 0 ? INFINITY : -INFINITY);
        out[i] = v;
        const double pe = v - prev;
        const double q = pe / delta + 0.5;
        int esc = 1;
        double cand = prev;
        if (q >= -max_m && q < max_m + 1.0) {
            const double mm = floor(q);
            cand = mm == 0.0 ? prev : prev + mm * delta;
            if (fabs(v - cand) <= eb) esc = 0;
        }
        prev = esc ? v : cand;
    }
}
