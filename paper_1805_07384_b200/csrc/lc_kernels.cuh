// lc_kernels.cuh -- parameter structs and kernel declarations shared by the
// .cu translation units and the C-ABI driver (lc_api.cu).
#pragma once
#include "lc_common.cuh"

// Host side: make a context's device current for one API call and restore
// the caller's current device on return (the C ABI never changes the calling
// thread's device as a side effect).
struct lc_ctx;
int lc_ctx_device(lc_ctx *ctx);

// lc_ctx_set_option keys (include/lossyckpt_b200.h)
#define LC_OPT_MAX_QUANT 0      // quantizer relaunches before the sequential fallback (default 64)
#define LC_OPT_MAX_REC 1        // decoder relaunches before the sequential fallback (default 64)
#define LC_OPT_INJECT_QUANT 2   // test hook: chunk whose predicted start is perturbed (-1 off)
#define LC_OPT_INJECT_REC 3     // test hook: the same in the decoder
#define LC_OPT_VERIFY 4         // 1: quantizer re-runs every chunk exactly (no certified skip)
#define LC_OPT_QUANT_RESUME 5   // 1 (default): a failed prediction resumes pass B; 0: full relaunch
// lc_ctx_get_stat keys
#define LC_STAT_QUANT_RELAUNCHES 0
#define LC_STAT_QUANT_SERIAL 1
#define LC_STAT_REC_RELAUNCHES 2
#define LC_STAT_REC_SERIAL 3
#define LC_STAT_QUANT_EXACT_CHUNKS 4
struct LcDeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit LcDeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~LcDeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

struct LcRangePart { double vmin, vmax, maxstep; int nonfinite; };

// Per-chunk prediction data written by pass A, read by pass B (SoA, [nchunks]).
struct LcChunkPred {
    int *kind;               // exclusive in-tile prefix map of the chunk (evaluation fields)
    double *B, *t0, *t1, *y;
    double *g0;              // guess of the chain value at the chunk start
};

// Bounds resolved on the device (lc_compress_auto_f64): the quantizer setup
// derived from the range pass without a host round trip.  skip != 0: nothing
// to quantize (status 10 non-finite, 11 2*eb overflow, 12 eb <= 0, 15 constant)
// and every later kernel of the call returns at once.
struct LcQuantDyn {
    LcQuant Q;
    double esc_thresh;
    double eb_abs, value_range, vmin, vmax, first_value;
    double rmax;             // (max |x| + eb)(1 + 2^-50): bounds every chain value (certification)
    int use_anchors;
    int skip;
    int status;
    int nonfinite;
};

struct LcQuantParams {
    const LcQuantDyn *dyn;   // non-null: Q / esc_thresh / use_anchors come from the device
    const double *x;
    uint64_t n;              // elements; codes cover positions 1..n-1
    LcQuant Q;
    double esc_thresh;       // |x_i - x_{i-1}| test for definite escapes
    int64_t first_chunk;     // relaunch start chunk (0 for a fresh run)
    double anchor_val;       // exact chain value at position first_chunk*L (x[0] read on device when 0)
    int64_t nchunks;         // total chunks ceil((n-1)/L)
    int64_t ntiles;          // tiles in this launch
    LcTileDesc *desc;
    unsigned int *tile_counter;
    uint32_t *hist;          // global histogram [nbins]
    uint32_t nbins;
    int count_hist;
    unsigned long long *first_bad;
    double *bad_end;         // per chunk: exact end value when its successor failed
    double *pe, *pe_rec;     // optional traces
    unsigned long long *nbig;      // codes >= the shared-memory histogram's range seen so far (lc_histw_kernel counts them)
    unsigned *maxcode;             // largest code produced so far (the codebook searches [0, maxcode] only)
    unsigned long long *timeline;  // optional: 8 globaltimer stamps per tile (profiling)
    // split-pass data
    int use_anchors;             // 0: no definite escape possible (range pass), anchor = launch anchor
    const long long *anc_in;     // [ntiles] last definite escape before each tile (>= launch anchor)
    long long *tile_last_esc;    // [ntiles] pass 0 output
    LcChunkPred pred;            // pass A -> pass B
    OffMap *tile_agg;            // [ntiles] pass A -> scan
    double *tile_S;              // [ntiles] pass A: certification slack of each warp tile
    double *tile_D;              // [ntiles + 1] scan -> pass B (offset at each tile start)
    long long inject_chunk;      // test hook: perturb this chunk's predicted start (fresh launch only), -1 off
    double rmax;                 // bound on |chain values| (from dyn)
    int verify;                  // 1: every chunk re-run exactly (no certified skip)
    unsigned long long *exact_count;   // chunks re-run exactly (diagnostic)
    // resume after a failed prediction without re-running pass A (lc_quant_wfix_kernel):
    int resume;                  // 0 first pass; 1 resume tile only; 2 the tiles after it
    int64_t first_tile;          // mode 2: first warp tile to process
    long long resume_chunk;      // first chunk whose predicted start was wrong
    const double *resume_start;  // its exact start (bad_end of its predecessor)
    double *resume_D0;           // mode 1 output: offset at the next tile start (NaN: resume impossible)
    double *tile_g0;             // [ntiles] pass A: guess of the chain value at each warp tile start
    double *sync_start;          // [nsync] exact chain value at every LC_SYNC_K-th element (v3 blocks)
    unsigned long long nsync;
};

// v2 blocks: a bit offset for every LC_SYNC_K-th symbol (a multiple of LC_L)
#define LC_SYNC_K 1024

struct LcCodebookOut {
    unsigned long long total_bits;
    unsigned long long n_esc;
    int max_len;
    int used;
    int status;              // 0 ok, 13 code length > 64
    int pad;
    unsigned long long stamp[6];   // phase timestamps (globaltimer, diagnostics)
};

struct LcStatsPart {
    double sum, comp;        // sum of squared errors (Neumaier: sum + comp)
    double maxabs, vmin, vmax, dev;
    int nonfinite;
    int pad;
};
__global__ void lc_stats_kernel(const double *__restrict__ a, const double *__restrict__ b, uint64_t n,
                                const double *__restrict__ pe, const double *__restrict__ pr,
                                LcStatsPart *__restrict__ parts);
__global__ void lc_stats_final_kernel(const LcStatsPart *__restrict__ parts, int np, LcStatsPart *__restrict__ out);

struct LcEncDesc {
    int st;
    int pad;
    unsigned long long agg_bits, agg_esc, incl_bits, incl_esc;
};

struct LcEncParams {
    const void *codes;       // u16 or u32 symbols [m]
    uint64_t m;              // number of symbols (n-1)
    const uint8_t *lengths;
    const unsigned long long *cw;
    uint32_t nbins;
    uint32_t *payload;       // words, zeroed
    const double *x;         // for escape values
    unsigned long long *esc_idx;
    double *esc_val;
    LcEncDesc *desc;
    unsigned int *tile_counter;
    uint64_t ntiles;
    const LcCodebookOut *cb; // device codebook summary (max_len <= 32: table path)
    const LcQuantDyn *dyn;   // device-resolved bounds (skip flag), may be null
    unsigned long long esc_cap;   // capacity of esc_idx / esc_val (host re-runs when short)
    unsigned long long *sync; // v2 sync table [ceil(m / LC_SYNC_K)] (bit offsets), may be null
    unsigned long long *sync_esc;   // v3: escape codes before every LC_SYNC_K-th symbol, may be null
    const unsigned long long *pending;   // quantizer's first failed chunk (~0: none); set: nothing to encode yet
};

__global__ void lc_range_kernel(const double *__restrict__ x, uint64_t n, LcRangePart *__restrict__ parts,
                                unsigned *__restrict__ done);
__global__ void lc_anchor_tiles_kernel(LcQuantParams P);
__global__ void lc_anchor_scan_kernel(const long long *__restrict__ last, long long *__restrict__ incoming,
                                      long long ntiles, long long launch_pos, const LcQuantDyn *dyn);
__global__ void lc_quant_setup_kernel(const LcRangePart *__restrict__ r, const double *__restrict__ x, uint64_t n,
                                      int eb_relative, double eb_param, uint32_t nbh, LcQuantDyn *d);
template <typename CodeT> __global__ void lc_quant_wa_kernel(LcQuantParams P, CodeT *__restrict__ codes);
template <typename CodeT, bool REC> __global__ void lc_quant_wfix_kernel(LcQuantParams P, CodeT *__restrict__ codes);
size_t lc_quantw_smem_bytes(int code_bytes);
int lc_decode_init_attrs();
size_t lc_quantw_fix_smem_bytes();
#define LC_WTILE (32 * LC_L)     // elements (codes) of one warp tile
#define LC_QW_TPB 128            // threads per CTA of the warp-tile quantizer kernels
__global__ void lc_map_scan_kernel(const OffMap *__restrict__ agg, double *__restrict__ tileD, long long ntiles,
                                   long long per, OffMap *gagg, int *gflag, const double *D0p);
// map scan launch: G co-resident CTAs of 1024 threads, `per` tiles per thread;
// scratch = LC_MAPSCAN_SCRATCH bytes (group aggregates + flags)
#define LC_MAPSCAN_MAXG 1024
#define LC_MAPSCAN_SCRATCH (LC_MAPSCAN_MAXG * (sizeof(OffMap) + sizeof(int)))
int lc_launch_map_scan(const OffMap *agg, double *tileD, long long ntiles, void *scratch, int sm_count,
                       cudaStream_t st, const double *D0p = nullptr);
template <typename CodeT> __global__ void lc_quant_serial_kernel(LcQuantParams P, CodeT *__restrict__ codes);
__global__ void lc_sync_starts_kernel(LcQuantParams P);
template <typename CodeT>
__global__ void lc_hist_kernel(const CodeT *__restrict__ codes, uint64_t m, uint32_t *__restrict__ hist, uint32_t nbins);
__global__ void lc_hist16_kernel(const uint16_t *__restrict__ codes, uint64_t m, uint32_t *__restrict__ hist,
                                 uint32_t nbins, const LcQuantDyn *dyn);
__global__ void lc_codebook_kernel(const uint32_t *__restrict__ hist, uint32_t nbins, uint8_t *__restrict__ lengths,
                                   unsigned long long *__restrict__ codes, unsigned long long *__restrict__ gkeys,
                                   unsigned long long *__restrict__ ifreq, int *__restrict__ parent, LcCodebookOut *out,
                                   const LcQuantDyn *dyn,
                                   const unsigned long long *pending, const unsigned *maxcode);
#define LC_HW_BINS 16384            // shared-memory bins of the wide-alphabet histogram pass (64 KB)
template <typename CodeT>
__global__ void lc_histw_kernel(const CodeT *__restrict__ codes, uint64_t m, uint32_t *__restrict__ hist, uint32_t nbins,
                                uint32_t lo, const unsigned long long *__restrict__ nbig,
                                const unsigned long long *__restrict__ pending, const LcQuantDyn *dyn);
__global__ void lc_zero_words_kernel(uint32_t *__restrict__ p, const LcCodebookOut *__restrict__ cb);
template <typename CodeT> __global__ void lc_encode_kernel(LcEncParams P);
size_t lc_codebook_smem_bytes();
size_t lc_encode_smem_bytes();
