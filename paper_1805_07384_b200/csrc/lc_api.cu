// lc_api.cu -- C ABI (include/lossyckpt_b200.h): contexts, compress and
// decompress drivers over the sm_100a kernels.
#include <chrono>
#include <mutex>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <string>
#include "../../include/lossyckpt_b200.h"

#include "lc_kernels.cuh"

int lc_decompress_impl2(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value,
                        const uint8_t *code_lengths, uint64_t n_lengths, const uint8_t *payload,
                        uint64_t payload_bytes, uint64_t payload_bits, const uint64_t *esc_idx,
                        const double *esc_val, uint64_t n_esc, int inputs_on_device, double *out,
                        int out_on_device, int64_t *esc_used, const uint64_t *sync, uint64_t n_sync,
                        const double *sync_starts = nullptr, const uint64_t *sync_esc = nullptr);

// ---------------------------------------------------------------------------

struct LcBuf {
    void *p = nullptr;
    size_t cap = 0;
};

struct lc_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t pev[12] = {};       // phase boundaries (lc_phase_ms)
    int last_kind = 0;              // 1 compress, 2 decompress
    bool debug_sync = false;        // LC_DEBUG_SYNC=1: sync + check after every launch
    bool timeline_on = false;       // LC_TIMELINE=1: per-tile phase stamps of the quantizer
    bool trace_on = false;          // LC_TRACE=1: an event + host timestamp after every launch
    cudaEvent_t tev[256] = {};
    const char *tname[256] = {};
    double thost[256] = {};
    int tn = 0;
    LcBuf timeline;
    int64_t timeline_tiles = 0;
    // lc_ctx_set_option knobs (tests / diagnostics)
    long long opt[8] = {64, 64, -1, -1, 0, 1, 0, 0};
    // per-context (hence per-device) launch state of the decoder (lc_decode.cu)
    int dec_state[40] = {};
    int quant_serial = 0;           // last compress finished with the sequential kernel
    uint32_t quant_relaunches = 0;
    unsigned long long quant_exact_chunks = 0;
    int quantw_occ[2][2] = {};      // resident CTAs per SM: [u32 codes][pass A, fix-up]
    void *mapscan_scratch = nullptr;
    uint64_t launches = 0;
    // scratch
    LcBuf xbuf, codes, hist, desc, counters, bad_end, pe, pe_rec, lengths, cw, gkeys, ifreq,
        parent, cbout, payload, esc_idx, esc_val, encdesc, range_parts, small, tiles;
    LcBuf st_b, st_pe, st_pr, st_parts, solver, sync;
    uint64_t nsync = 0;                 // v2 sync offsets of the last compress
    // last lc_range_f64 on device data (lets compress skip the anchor pass)
    const void *rng_ptr = nullptr;
    uint64_t rng_n = 0;
    double rng_maxstep = INFINITY;
    void *pinned = nullptr;         // small pinned staging
    // last compress result
    uint64_t n = 0;
    uint32_t nbins = 0;
    int code_bytes = 2;
    int record = 0;
    LcCodebookOut cb{};
    // decompress scratch (lc_decode.cu)
    LcBuf dec[10];     // payload, lengths, esc idx, esc val, out, codes, tables, sync, aux, aux2
};

int lc_fail(lc_ctx *ctx, cudaError_t e, const char *what, const char *file, int line)
{
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    if (ctx) ctx->err = buf;
    return 20;
}

cudaError_t lc_reserve(LcBuf &b, size_t bytes)
{
    if (bytes <= b.cap && b.p) return cudaSuccess;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    size_t cap = bytes < 256 ? 256 : bytes + bytes / 8;
    cudaError_t e = cudaMalloc(&b.p, cap);
    if (e == cudaSuccess) b.cap = cap;
    return e;
}

cudaStream_t lc_stream(lc_ctx *ctx) { return ctx->stream; }
int lc_sm_count(lc_ctx *ctx) { return ctx->sm_count; }
void *lc_pinned(lc_ctx *ctx) { return ctx->pinned; }
void *lc_solver_scratch(lc_ctx *ctx, size_t bytes)
{
    return lc_reserve(ctx->solver, bytes) == cudaSuccess ? ctx->solver.p : nullptr;
}
void lc_set_err(lc_ctx *ctx, const char *msg) { ctx->err = msg; }
LcBuf *lc_dec_bufs(lc_ctx *ctx) { return ctx->dec; }
cudaEvent_t lc_phase_ev(lc_ctx *ctx, int i) { return ctx->pev[i]; }
void lc_count_launch(lc_ctx *ctx, int k) { ctx->launches += k; }
long long lc_opt(lc_ctx *ctx, int key) { return (key >= 0 && key < 8) ? ctx->opt[key] : 0; }
int *lc_dec_state(lc_ctx *ctx) { return ctx->dec_state; }

int lc_ctx_device(lc_ctx *ctx) { return ctx->device; }
void lc_set_kind(lc_ctx *ctx, int k) { ctx->last_kind = k; }

static double lc_host_us()
{
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void lc_trace_mark(lc_ctx *ctx, const char *what)
{
    if (!ctx->trace_on || ctx->tn >= 256) return;
    if (!ctx->tev[ctx->tn]) cudaEventCreate(&ctx->tev[ctx->tn]);
    ctx->thost[ctx->tn] = lc_host_us();
    ctx->tname[ctx->tn] = what;
    cudaEventRecord(ctx->tev[ctx->tn], ctx->stream);
    ++ctx->tn;
}

int lc_debug_check(lc_ctx *ctx, const char *what, const char *file, int line)
{
    lc_trace_mark(ctx, what);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && ctx->debug_sync) {
        const bool log = getenv("LC_DEBUG_LOG") != nullptr;       // LC_DEBUG_LOG=1: name every checked launch (stderr)
        if (log) fprintf(stderr, "[lc] %s:%d %s ...", file, line, what);
        e = cudaStreamSynchronize(ctx->stream);
        if (log) fprintf(stderr, " %s\n", cudaGetErrorName(e));
    }
    if (e != cudaSuccess) return lc_fail(ctx, e, what, file, line);
    return 0;
}

extern "C" {

int lc_ctx_create(lc_ctx **out, int device, void *stream)
{
    LcDeviceGuard guard(device);
    lc_ctx *ctx = new lc_ctx();
    ctx->device = device;
    *out = nullptr;
    const char *dbg = getenv("LC_DEBUG_SYNC");
    ctx->debug_sync = dbg && dbg[0] == '1';
    const char *tlv = getenv("LC_TIMELINE");
    ctx->timeline_on = tlv && tlv[0] == '1';
    const char *trv = getenv("LC_TRACE");
    ctx->trace_on = trv && trv[0] == '1';
    if (!guard.ok) LC_CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop;
    LC_CUDA_OK(cudaGetDeviceProperties(&prop, device));
    ctx->sm_count = prop.multiProcessorCount;
    // NULL selects the legacy default stream (ordered with torch's default stream)
    ctx->stream = (cudaStream_t)stream;
    LC_CUDA_OK(cudaEventCreate(&ctx->ev0));
    LC_CUDA_OK(cudaEventCreate(&ctx->ev1));
    for (int i = 0; i < 12; ++i) LC_CUDA_OK(cudaEventCreate(&ctx->pev[i]));
    LC_CUDA_OK(cudaMallocHost(&ctx->pinned, 4096));
    {
        const size_t q16 = lc_quantw_smem_bytes(2), q32 = lc_quantw_smem_bytes(4), qf = lc_quantw_fix_smem_bytes();
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wa_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q16));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wa_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q32));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wfix_kernel<uint16_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qf));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wfix_kernel<uint32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qf));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wfix_kernel<uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qf));
        LC_CUDA_OK(cudaFuncSetAttribute(lc_quant_wfix_kernel<uint32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qf));
        // persistent grids sized to one resident wave
        LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->quantw_occ[0][0], lc_quant_wa_kernel<uint16_t>, LC_QW_TPB, q16));
        LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->quantw_occ[1][0], lc_quant_wa_kernel<uint32_t>, LC_QW_TPB, q32));
        LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->quantw_occ[0][1], lc_quant_wfix_kernel<uint16_t, false>, LC_QW_TPB, qf));
        LC_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->quantw_occ[1][1], lc_quant_wfix_kernel<uint32_t, false>, LC_QW_TPB, qf));
        for (auto &a2 : ctx->quantw_occ)
            for (int &o : a2) o = o > 0 ? o : 1;
    }
    LC_CUDA_OK((cudaError_t)lc_decode_init_attrs());
    LC_CUDA_OK(cudaFuncSetAttribute(lc_histw_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(LC_HW_BINS * sizeof(uint32_t))));
    LC_CUDA_OK(cudaFuncSetAttribute(lc_histw_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(LC_HW_BINS * sizeof(uint32_t))));
    LC_CUDA_OK(cudaFuncSetAttribute(lc_codebook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)lc_codebook_smem_bytes()));
    LC_CUDA_OK(cudaFuncSetAttribute(lc_encode_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)lc_encode_smem_bytes()));
    LC_CUDA_OK(cudaFuncSetAttribute(lc_encode_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)lc_encode_smem_bytes()));
    *out = ctx;
    return 0;
}

void lc_ctx_destroy(lc_ctx *ctx)
{
    if (!ctx) return;
    LcDeviceGuard guard(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    LcBuf *bufs[] = {&ctx->xbuf, &ctx->codes, &ctx->hist, &ctx->desc, &ctx->counters, &ctx->bad_end,
                     &ctx->pe, &ctx->pe_rec, &ctx->lengths, &ctx->cw, &ctx->gkeys, &ctx->ifreq,
                     &ctx->parent, &ctx->cbout, &ctx->payload, &ctx->esc_idx, &ctx->esc_val,
                     &ctx->encdesc, &ctx->range_parts, &ctx->small, &ctx->tiles, &ctx->dec[0], &ctx->dec[1],
                     &ctx->dec[2], &ctx->dec[3], &ctx->dec[4], &ctx->dec[5], &ctx->dec[6],
                     &ctx->dec[7], &ctx->dec[8], &ctx->dec[9], &ctx->st_b, &ctx->st_pe, &ctx->st_pr,
                     &ctx->st_parts, &ctx->solver, &ctx->sync};
    for (LcBuf *b : bufs)
        if (b->p) cudaFree(b->p);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (int i = 0; i < 12; ++i)
        if (ctx->pev[i]) cudaEventDestroy(ctx->pev[i]);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *lc_last_error(lc_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

double lc_last_device_ms(lc_ctx *ctx)
{
    float ms = -1.0f;
    if (cudaEventSynchronize(ctx->ev1) != cudaSuccess) return -1.0;   // the end event may still be queued
    if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) != cudaSuccess) return -1.0;
    return ms;
}

static const double *lc_device_input(lc_ctx *ctx, const double *x, uint64_t n, int on_device, int *rc)
{
    *rc = 0;
    if (on_device) return x;
    cudaError_t e = lc_reserve(ctx->xbuf, n * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->xbuf.p, x, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) { *rc = lc_fail(ctx, e, "input H2D", __FILE__, __LINE__); return nullptr; }
    return (const double *)ctx->xbuf.p;
}

int lc_range_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device, double *vmin, double *vmax,
                 int *nonfinite)
{
    if (!ctx || n == 0) return 12;
    LcDeviceGuard guard(ctx->device);
    int rc;
    const double *dx = lc_device_input(ctx, x, n, x_on_device, &rc);
    if (rc) return rc;
    int nb = (int)((n + 255) / 256);
    if (nb > 4 * ctx->sm_count) nb = 4 * ctx->sm_count;
    LC_CUDA_OK(lc_reserve(ctx->range_parts, sizeof(LcRangePart) * (nb + 1) + 16));
    LcRangePart *parts = (LcRangePart *)ctx->range_parts.p;
    unsigned *done = (unsigned *)(parts + nb + 1);
    LC_CUDA_OK(cudaMemsetAsync(done, 0, sizeof(unsigned), ctx->stream));
    lc_range_kernel<<<nb, 256, 0, ctx->stream>>>(dx, n, parts, done);
    ctx->launches += 1;
    { int _rc = lc_debug_check(ctx, "lc_range_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    LcRangePart *h = (LcRangePart *)ctx->pinned;
    LC_CUDA_OK(cudaMemcpyAsync(h, parts + nb, sizeof(LcRangePart), cudaMemcpyDeviceToHost, ctx->stream));
    LC_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *vmin = h->vmin;
    *vmax = h->vmax;
    *nonfinite = h->nonfinite;
    ctx->rng_ptr = x_on_device ? (const void *)x : nullptr;
    ctx->rng_n = n;
    ctx->rng_maxstep = h->maxstep;
    return 0;
}

int lc_error_stats_f64(lc_ctx *ctx, const double *original, const double *recon, uint64_t n, int on_device,
                       const double *pe, const double *pe_rec, lc_stats *out)
{
    if (!ctx || !out || n == 0) return 12;
    LcDeviceGuard guard(ctx->device);
    cudaStream_t st = ctx->stream;
    int rc;
    const double *da = lc_device_input(ctx, original, n, on_device, &rc);
    if (rc) return rc;
    auto stage = [&](LcBuf &buf, const double *h, uint64_t cnt) -> const double * {
        if (on_device || !h) return h;
        if (lc_reserve(buf, cnt * sizeof(double)) != cudaSuccess) return nullptr;
        if (cudaMemcpyAsync(buf.p, h, cnt * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) return nullptr;
        return (const double *)buf.p;
    };
    const double *db = stage(ctx->st_b, recon, n);
    const bool with_pe = pe && pe_rec && n > 1;
    const double *dpe = with_pe ? stage(ctx->st_pe, pe, n - 1) : nullptr;
    const double *dpr = with_pe ? stage(ctx->st_pr, pe_rec, n - 1) : nullptr;
    if (!db || (with_pe && (!dpe || !dpr))) return lc_fail(ctx, cudaErrorMemoryAllocation, "stats H2D", __FILE__, __LINE__);
    int nb = (int)((n + 255) / 256);
    if (nb > 4 * ctx->sm_count) nb = 4 * ctx->sm_count;
    LC_CUDA_OK(lc_reserve(ctx->st_parts, sizeof(LcStatsPart) * (nb + 1)));
    LcStatsPart *parts = (LcStatsPart *)ctx->st_parts.p;
    lc_stats_kernel<<<nb, 256, 0, st>>>(da, db, n, dpe, dpr, parts);
    lc_stats_final_kernel<<<1, 1, 0, st>>>(parts, nb, parts + nb);
    ctx->launches += 2;
    { int _rc = lc_debug_check(ctx, "lc_stats_final_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    LcStatsPart *h = (LcStatsPart *)ctx->pinned;
    LC_CUDA_OK(cudaMemcpyAsync(h, parts + nb, sizeof(LcStatsPart), cudaMemcpyDeviceToHost, st));
    LC_CUDA_OK(cudaStreamSynchronize(st));
    out->sum_sq_err = h->sum + h->comp;
    out->max_abs_err = h->maxabs;
    out->vmin = h->vmin;
    out->vmax = h->vmax;
    out->max_identity_dev = with_pe ? h->dev : -1.0;
    out->nonfinite = h->nonfinite;
    return 0;
}

}  // extern "C"

// dyn (device) non-null: the bounds were resolved on the device by
// lc_quant_setup_kernel (eb_abs is unused); *hdyn receives them with the one
// readback and a non-zero hdyn->status is returned without results.
template <typename CodeT>
static int lc_compress_t(lc_ctx *ctx, const double *dx, uint64_t n, double eb_abs, uint32_t nbh, int record,
                         lc_result *res, const LcQuantDyn *dyn = nullptr, LcQuantDyn *hdyn = nullptr)
{
    cudaStream_t st = ctx->stream;
    const uint32_t nbins = 2u * nbh;
    const int64_t nchunks = (int64_t)((n - 1 + LC_L - 1) / LC_L);
    const int64_t ntiles = (nchunks + 31) / 32;          // warp tiles (lc_quantw.cu)
    const uint64_t m = n - 1;
    LC_CUDA_OK(lc_reserve(ctx->codes, m * sizeof(CodeT)));
    LC_CUDA_OK(lc_reserve(ctx->hist, nbins * sizeof(uint32_t)));
    LC_CUDA_OK(lc_reserve(ctx->counters, 128));
    LC_CUDA_OK(lc_reserve(ctx->bad_end, nchunks * sizeof(double)));
    if (record) {
        LC_CUDA_OK(lc_reserve(ctx->pe, m * sizeof(double)));
        LC_CUDA_OK(lc_reserve(ctx->pe_rec, m * sizeof(double)));
    }
    unsigned int *tile_counter = (unsigned int *)ctx->counters.p;
    unsigned long long *first_bad = (unsigned long long *)((char *)ctx->counters.p + 16);
    unsigned long long *exact_count = (unsigned long long *)((char *)ctx->counters.p + 32);
    unsigned long long *nbig = (unsigned long long *)((char *)ctx->counters.p + 64);
    unsigned *maxcode = (unsigned *)((char *)ctx->counters.p + 72);

    LcQuantParams P;
    memset(&P, 0, sizeof P);
    P.dyn = dyn;
    P.x = dx;
    P.n = n;
    P.Q.delta = 2.0 * eb_abs;          // host bounds are only used when dyn is null (never in practice)
    P.Q.eb = eb_abs;
    P.Q.max_m = (double)(nbh - 1);
    P.Q.max_m1 = P.Q.max_m + 1.0;
    P.Q.inv = 1.0 / P.Q.delta;
    {   // decision margin of lc_step_nb: T = 2^e >= 2^-50 (max_m + 2)
        int e2;
        frexp(P.Q.max_m + 2.0, &e2);
        P.Q.cert = 0.5 - ldexp(1.0, e2 - 50);
    }
    P.esc_thresh = (double)nbh * P.Q.delta * (1.0 + 0x1p-40);
    P.rmax = INFINITY;                 // no range known: certification off
    P.first_chunk = 0;
    P.anchor_val = 0.0;
    P.nchunks = nchunks;
    P.tile_counter = tile_counter;
    P.hist = (uint32_t *)ctx->hist.p;
    P.nbins = nbins;
    P.count_hist = 1;
    P.first_bad = first_bad;
    P.bad_end = (double *)ctx->bad_end.p;
    P.pe = record ? (double *)ctx->pe.p : nullptr;
    P.pe_rec = record ? (double *)ctx->pe_rec.p : nullptr;
    P.verify = ctx->opt[LC_OPT_VERIFY] ? 1 : 0;
    P.exact_count = exact_count;
    P.nbig = nbig;
    P.maxcode = maxcode;
    P.resume = 0;
    P.first_tile = 0;
    P.resume_chunk = -1;
    P.resume_start = nullptr;
    P.resume_D0 = (double *)((char *)ctx->counters.p + 48);
    P.timeline = nullptr;
    if (ctx->timeline_on) {                    // LC_TIMELINE=1: per-tile globaltimer stamps (diagnostics)
        LC_CUDA_OK(lc_reserve(ctx->timeline, ntiles * 128));
        LC_CUDA_OK(cudaMemsetAsync(ctx->timeline.p, 0, ntiles * 128, st));
        P.timeline = (unsigned long long *)ctx->timeline.p;
        ctx->timeline_tiles = ntiles;
    }
    CodeT *codes = (CodeT *)ctx->codes.p;

    LC_CUDA_OK(cudaMemsetAsync(P.hist, 0, nbins * sizeof(uint32_t), st));
    LC_CUDA_OK(cudaMemsetAsync(exact_count, 0, 8, st));
    LC_CUDA_OK(cudaMemsetAsync(nbig, 0, 16, st));            // nbig and maxcode

    unsigned long long *hbad = (unsigned long long *)ctx->pinned;
    LcCodebookOut *hcb = (LcCodebookOut *)((char *)ctx->pinned + 64);
    unsigned long long *hexact = (unsigned long long *)((char *)ctx->pinned + 192);
    uint32_t relaunches = 0;
    bool full = false;                                   // a full quantizer relaunch happened
    ctx->quant_serial = 0;
    P.inject_chunk = ctx->opt[LC_OPT_INJECT_QUANT];
    LC_CUDA_OK(cudaEventRecord(ctx->pev[1], st));
    LC_CUDA_OK(lc_reserve(ctx->tiles, (size_t)(ntiles + 1) * (2 * sizeof(long long) + sizeof(OffMap) + 3 * sizeof(double))
                                          + LC_MAPSCAN_SCRATCH + 256));
    {
        char *pp = (char *)ctx->tiles.p;
        P.tile_agg = (OffMap *)pp;               pp += (ntiles + 1) * sizeof(OffMap);
        P.tile_D = (double *)pp;                 pp += (ntiles + 1) * sizeof(double);
        P.tile_S = (double *)pp;                 pp += (ntiles + 1) * sizeof(double);
        P.tile_g0 = (double *)pp;                pp += (ntiles + 1) * sizeof(double);
        P.tile_last_esc = (long long *)pp;       pp += (ntiles + 1) * sizeof(long long);
        P.anc_in = (const long long *)pp;        pp += (ntiles + 1) * sizeof(long long);
        ctx->mapscan_scratch = (void *)(((uintptr_t)pp + 63) & ~(uintptr_t)63);
    }
    long long *anc_in = (long long *)P.anc_in;
    P.use_anchors = 1;                                   // with dyn: the device decides
    const size_t qsmem = lc_quantw_smem_bytes(sizeof(CodeT)), fsmem = lc_quantw_fix_smem_bytes();
    const int ga = 3 * ctx->sm_count;
    const int *occ = ctx->quantw_occ[sizeof(CodeT) == 2 ? 0 : 1];
    auto quant_launch = [&]() -> int {
        P.ntiles = (nchunks - P.first_chunk + 31) / 32;
        LC_CUDA_OK(cudaMemsetAsync(first_bad, 0xff, 8, st));
        if (P.use_anchors) {
            lc_anchor_tiles_kernel<<<(int)((P.ntiles + 7) / 8 < ga ? (P.ntiles + 7) / 8 : ga), LC_TPB, 0, st>>>(P);
            { int _rc = lc_debug_check(ctx, "lc_anchor_tiles_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
            lc_anchor_scan_kernel<<<1, 1024, 0, st>>>(P.tile_last_esc, anc_in, P.ntiles, P.first_chunk * LC_L, dyn);
            { int _rc = lc_debug_check(ctx, "lc_anchor_scan_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
            ctx->launches += 2;
        }
        const long long wcta = (P.ntiles + LC_QW_TPB / 32 - 1) / (LC_QW_TPB / 32);
        LC_CUDA_OK(cudaMemsetAsync(tile_counter, 0, 4, st));
        const long long ga2 = (long long)occ[0] * ctx->sm_count, gf = (long long)occ[1] * ctx->sm_count;
        lc_quant_wa_kernel<CodeT><<<(int)(wcta < ga2 ? wcta : ga2), LC_QW_TPB, qsmem, st>>>(P, codes);
        { int _rc = lc_debug_check(ctx, "lc_quant_wa_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        LC_CUDA_OK((cudaError_t)lc_launch_map_scan(P.tile_agg, P.tile_D, P.ntiles, ctx->mapscan_scratch,
                                                   ctx->sm_count, st));
        { int _rc = lc_debug_check(ctx, "lc_map_scan_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        if (P.pe) lc_quant_wfix_kernel<CodeT, true><<<(int)(wcta < gf ? wcta : gf), LC_QW_TPB, fsmem, st>>>(P, codes);
        else lc_quant_wfix_kernel<CodeT, false><<<(int)(wcta < gf ? wcta : gf), LC_QW_TPB, fsmem, st>>>(P, codes);
        { int _rc = lc_debug_check(ctx, "lc_quant_wfix_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        lc_sync_starts_kernel<<<(int)((P.ntiles + 255) / 256 < 2 * ctx->sm_count ? (P.ntiles + 255) / 256
                                                                                : 2 * ctx->sm_count), 256, 0, st>>>(P);
        ctx->launches += 4;
        return 0;
    };

    // codebook + encoder buffers: the payload is at most ceil(log2(nbins)) bits per
    // symbol (a fixed-length code is never shorter than the Huffman code), so it is
    // sized before the codebook is known; escapes use the capacity of the last call
    // and are re-gathered when short (the host sees the count after the one sync).
    int lg = 1;
    while ((1ull << lg) < nbins) ++lg;
    const uint64_t words_cap = (m * (uint64_t)lg + 31) / 32 + 2;
    LC_CUDA_OK(lc_reserve(ctx->payload, words_cap * 4));
    LC_CUDA_OK(lc_reserve(ctx->esc_idx, 64 * 8));
    LC_CUDA_OK(lc_reserve(ctx->esc_val, 64 * 8));
    LC_CUDA_OK(lc_reserve(ctx->lengths, nbins));
    LC_CUDA_OK(lc_reserve(ctx->cw, nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->gkeys, 3 * (size_t)nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->ifreq, (size_t)nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->parent, 2 * (size_t)nbins * sizeof(int)));
    LC_CUDA_OK(lc_reserve(ctx->cbout, sizeof(LcCodebookOut)));
    LcCodebookOut *cbo = (LcCodebookOut *)ctx->cbout.p;
    const uint64_t etiles = (m + LC_TILE - 1) / LC_TILE;
    LC_CUDA_OK(lc_reserve(ctx->encdesc, etiles * sizeof(LcEncDesc)));
    ctx->nsync = (m + LC_SYNC_K - 1) / LC_SYNC_K;
    // sync table of every compress: bit offsets, exact chain values and escape
    // counts at every LC_SYNC_K-th symbol (v2 blocks use the offsets, v3 all three)
    LC_CUDA_OK(lc_reserve(ctx->sync, (ctx->nsync + 1) * 24));
    P.sync_start = (double *)ctx->sync.p + (ctx->nsync + 1);
    P.nsync = ctx->nsync;
    LcEncParams E;
    E.codes = codes;
    E.m = m;
    E.lengths = (const uint8_t *)ctx->lengths.p;
    E.cw = (const unsigned long long *)ctx->cw.p;
    E.nbins = nbins;
    E.payload = (uint32_t *)ctx->payload.p;
    E.x = dx;
    E.desc = (LcEncDesc *)ctx->encdesc.p;
    E.tile_counter = tile_counter;
    E.ntiles = etiles;
    E.cb = cbo;
    E.sync = (unsigned long long *)ctx->sync.p;
    E.sync_esc = (unsigned long long *)ctx->sync.p + 2 * (ctx->nsync + 1);
    E.dyn = dyn;
    E.pending = first_bad;
    const int egrid = (int)(etiles < (uint64_t)(4 * ctx->sm_count) ? etiles : 4 * ctx->sm_count);
    auto histw_launch = [&]() -> int {                   // codes beyond pass A's shared-memory bins
        if (nbins <= LC_HBINS_B) return 0;
        lc_histw_kernel<CodeT><<<2 * ctx->sm_count, 512, LC_HW_BINS * sizeof(uint32_t), st>>>(
            codes, m, P.hist, nbins, LC_HBINS_B, nbig, first_bad, dyn);
        { int _rc = lc_debug_check(ctx, "lc_histw_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        ctx->launches += 1;
        return 0;
    };
    auto codebook_launch = [&]() -> int {
        LC_CUDA_OK(cudaEventRecord(ctx->pev[2], st));
        lc_codebook_kernel<<<1, 1024, lc_codebook_smem_bytes(), st>>>(
            P.hist, nbins, (uint8_t *)ctx->lengths.p, (unsigned long long *)ctx->cw.p,
            (unsigned long long *)ctx->gkeys.p, (unsigned long long *)ctx->ifreq.p, (int *)ctx->parent.p, cbo, dyn,
            first_bad, full ? nullptr : maxcode);
        { int _rc = lc_debug_check(ctx, "lc_codebook_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        LC_CUDA_OK(cudaEventRecord(ctx->pev[3], st));
        ctx->launches += 1;
        return 0;
    };
    auto encode_launch = [&]() -> int {
        E.esc_idx = (unsigned long long *)ctx->esc_idx.p;
        E.esc_val = (double *)ctx->esc_val.p;
        E.esc_cap = ctx->esc_idx.cap / 8;
        lc_zero_words_kernel<<<2 * ctx->sm_count, 256, 0, st>>>((uint32_t *)ctx->payload.p, cbo);
        LC_CUDA_OK(cudaMemsetAsync(ctx->encdesc.p, 0, etiles * sizeof(LcEncDesc), st));
        LC_CUDA_OK(cudaMemsetAsync(ctx->counters.p, 0, 16, st));
        lc_encode_kernel<CodeT><<<egrid, LC_TPB + 32, lc_encode_smem_bytes(), st>>>(E);
        { int _rc = lc_debug_check(ctx, "lc_encode_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        ctx->launches += 2;
        LC_CUDA_OK(cudaEventRecord(ctx->pev[4], st));
        return 0;
    };
    auto readback = [&]() -> int {                       // the one host round trip
        LC_CUDA_OK(cudaMemcpyAsync(hbad, first_bad, 8, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaMemcpyAsync(hexact, exact_count, 8, cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaMemcpyAsync(hcb, cbo, sizeof(LcCodebookOut), cudaMemcpyDeviceToHost, st));
        if (dyn) LC_CUDA_OK(cudaMemcpyAsync(hdyn, dyn, sizeof(LcQuantDyn), cudaMemcpyDeviceToHost, st));
        LC_CUDA_OK(cudaStreamSynchronize(st));
        return 0;
    };

    // common path: quantize, codebook and encode back to back, one sync
    { int _rc = quant_launch(); if (_rc) return _rc; }
    { int _rc = histw_launch(); if (_rc) return _rc; }
    { int _rc = codebook_launch(); if (_rc) return _rc; }
    { int _rc = encode_launch(); if (_rc) return _rc; }
    { int _rc = readback(); if (_rc) return _rc; }
    if (dyn && hdyn->status) return hdyn->status;        // non-finite / constant / bad bound: no results
    if (dyn && hdyn->rmax < 0x1p-960) {
        // every value below 2^-960: ulps are subnormal and the offset-map arithmetic is not exact
        // (predicted chunk and tile starts can be an ulp off), so the sequential exact chain does
        // the whole vector; it also writes the v3 sync starts itself
        P.first_chunk = 0;
        P.inject_chunk = -1;
        ctx->quant_serial = 1;
        LC_CUDA_OK(cudaMemsetAsync(first_bad, 0xff, 8, st));
        lc_quant_serial_kernel<CodeT><<<1, 32, 0, st>>>(P, codes);
        { int _rc = lc_debug_check(ctx, "lc_quant_serial_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        ctx->launches += 1;
        relaunches = 1;
        full = true;
        *hbad = ~0ULL;
    }
    if (*hbad != ~0ULL) {
        // a chunk prediction failed.  Resume (default): pass A's results stand, the
        // chunks from the first bad one to the end of its warp tile are re-run from
        // its exact start, the remaining tiles get new offsets from a map scan and
        // go through pass B again (lc_quant_wfix_kernel modes 1 and 2; the
        // histogram is kept exact by pass B's per-code updates).  A full relaunch
        // from the first bad chunk (anchor = the exact end of its predecessor) is
        // the fallback when the new offset is not representable, or when resuming
        // is switched off (LC_OPT_QUANT_RESUME = 0).
        double *hD0 = (double *)((char *)ctx->pinned + 200);
        for (;;) {
            const unsigned long long fb = *hbad;
            if (fb == ~0ULL) break;
            ++relaunches;
            P.inject_chunk = -1;
            if (ctx->opt[LC_OPT_QUANT_RESUME] && (long long)relaunches <= ctx->opt[LC_OPT_MAX_QUANT]) {
                const long long wf = ((long long)fb - P.first_chunk) / 32;
                const long long wcta = (P.ntiles + LC_QW_TPB / 32 - 1) / (LC_QW_TPB / 32);
                const long long gf = (long long)occ[1] * ctx->sm_count;
                P.resume = 1;
                P.resume_chunk = (long long)fb;
                P.resume_start = P.bad_end + (fb - 1);
                LC_CUDA_OK(cudaMemsetAsync(first_bad, 0xff, 8, st));
                if (P.pe) lc_quant_wfix_kernel<CodeT, true><<<1, 32, fsmem, st>>>(P, codes);
                else lc_quant_wfix_kernel<CodeT, false><<<1, 32, fsmem, st>>>(P, codes);
                ctx->launches += 1;
                { int _rc = lc_debug_check(ctx, "lc_quant_wfix_kernel (resume 1)", __FILE__, __LINE__); if (_rc) return _rc; }
                if (wf + 1 < P.ntiles) {
                    LC_CUDA_OK((cudaError_t)lc_launch_map_scan(P.tile_agg + wf + 1, P.tile_D + wf + 1,
                                                               P.ntiles - wf - 1, ctx->mapscan_scratch,
                                                               ctx->sm_count, st, P.resume_D0));
                    { int _rc = lc_debug_check(ctx, "lc_map_scan_kernel (resume)", __FILE__, __LINE__); if (_rc) return _rc; }
                    P.resume = 2;
                    P.first_tile = wf + 1;
                    if (P.pe) lc_quant_wfix_kernel<CodeT, true><<<(int)(wcta < gf ? wcta : gf), LC_QW_TPB, fsmem, st>>>(P, codes);
                    else lc_quant_wfix_kernel<CodeT, false><<<(int)(wcta < gf ? wcta : gf), LC_QW_TPB, fsmem, st>>>(P, codes);
                    ctx->launches += 2;
                }
                { int _rc = lc_debug_check(ctx, "lc_quant_wfix_kernel (resume)", __FILE__, __LINE__); if (_rc) return _rc; }
                P.resume = 0;
                P.first_tile = 0;
                lc_sync_starts_kernel<<<(int)((P.ntiles + 255) / 256 < 2 * ctx->sm_count ? (P.ntiles + 255) / 256
                                                                                        : 2 * ctx->sm_count), 256, 0, st>>>(P);
                ctx->launches += 1;
                LC_CUDA_OK(cudaMemcpyAsync(hbad, first_bad, 8, cudaMemcpyDeviceToHost, st));
                LC_CUDA_OK(cudaMemcpyAsync(hD0, P.resume_D0, 8, cudaMemcpyDeviceToHost, st));
                LC_CUDA_OK(cudaStreamSynchronize(st));
                if (*hD0 == *hD0 || *hbad != fb) continue;   // resumed (or the next failure is elsewhere)
            }
            full = true;
            // relaunch from the start of the failing chunk's warp tile (launches stay
            // tile aligned, so v3 sync starts map onto warp tiles): its exact start
            // is the failing chunk's exact start, or the tile's sync start (before
            // the first failure every predicted start is exact)
            const long long fa = P.first_chunk + (((long long)fb - P.first_chunk) / 32) * 32;
            double anchor;
            if (fa == (long long)fb)
                LC_CUDA_OK(cudaMemcpy(&anchor, P.bad_end + (fb - 1), sizeof(double), cudaMemcpyDeviceToHost));
            else
                LC_CUDA_OK(cudaMemcpy(&anchor, P.sync_start + fa / 32, sizeof(double), cudaMemcpyDeviceToHost));
            if (!isfinite(anchor)) {
                // a prediction failed before any exact start was known (the offset
                // look-back gave no finite value): restart this launch sequentially
                relaunches = (uint32_t)ctx->opt[LC_OPT_MAX_QUANT] + 1;
            } else {
                P.first_chunk = (int64_t)fa;
                P.anchor_val = anchor;
            }
            P.inject_chunk = -1;
            if ((long long)relaunches > ctx->opt[LC_OPT_MAX_QUANT]) {   // pathological input: exact serial chain
                ctx->quant_serial = 1;
                LC_CUDA_OK(cudaMemsetAsync(first_bad, 0xff, 8, st));    // nothing pending after the exact chain
                lc_quant_serial_kernel<CodeT><<<1, 32, 0, st>>>(P, codes);
                { int _rc = lc_debug_check(ctx, "lc_quant_serial_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
                ctx->launches += 1;
                break;
            }
            { int _rc = quant_launch(); if (_rc) return _rc; }
            LC_CUDA_OK(cudaMemcpyAsync(hbad, first_bad, 8, cudaMemcpyDeviceToHost, st));
            LC_CUDA_OK(cudaStreamSynchronize(st));
        }
    }
    if (relaunches) {
        if (full) {                       // a full relaunch counted its chunks' codes again: recount
        LC_CUDA_OK(cudaMemsetAsync(P.hist, 0, nbins * sizeof(uint32_t), st));
        if (sizeof(CodeT) == 2)      // streaming pass with packed per-thread counters for codes 1..16
            lc_hist16_kernel<<<4 * ctx->sm_count, 256, 0, st>>>(reinterpret_cast<const uint16_t *>(codes), m, P.hist,
                                                               nbins, nullptr);
        else
            lc_hist_kernel<CodeT><<<4 * ctx->sm_count, 256, 0, st>>>(codes, m, P.hist, nbins);
        { int _rc = lc_debug_check(ctx, "lc_hist_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
        ctx->launches += 1;
        LC_CUDA_OK(cudaMemsetAsync(nbig, 0, 8, st));     // the recount covered every bin
        }
        { int _rc = histw_launch(); if (_rc) return _rc; }
        { int _rc = codebook_launch(); if (_rc) return _rc; }
        { int _rc = encode_launch(); if (_rc) return _rc; }
        { int _rc = readback(); if (_rc) return _rc; }
    }
    ctx->quant_exact_chunks = *hexact;
    ctx->cb = *hcb;
    if (ctx->cb.status) {
        ctx->err = "code length exceeds 64 bits";
        return ctx->cb.status;
    }
    if (ctx->cb.n_esc > ctx->esc_idx.cap / 8) {          // more escapes than the last call: re-gather
        LC_CUDA_OK(lc_reserve(ctx->esc_idx, (ctx->cb.n_esc + 1) * 8));
        LC_CUDA_OK(lc_reserve(ctx->esc_val, (ctx->cb.n_esc + 1) * 8));
        { int _rc = encode_launch(); if (_rc) return _rc; }
        { int _rc = readback(); if (_rc) return _rc; }
    }
    LC_CUDA_OK(cudaEventRecord(ctx->ev1, st));
    ctx->last_kind = 1;

    ctx->n = n;
    ctx->nbins = nbins;
    ctx->code_bytes = sizeof(CodeT);
    ctx->record = record;
    res->n = n;
    res->payload_bits = ctx->cb.total_bits;
    res->payload_bytes = (ctx->cb.total_bits + 7) / 8;
    res->n_esc = ctx->cb.n_esc;
    res->n_symbols = nbins;
    res->max_len = (uint32_t)ctx->cb.max_len;
    res->used_symbols = (uint32_t)ctx->cb.used;
    res->relaunches = relaunches;
    ctx->quant_relaunches = relaunches;
    return 0;
}

extern "C" {

int lc_compress_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device, double eb_abs,
                    uint32_t n_bins_half, int record_traces, lc_result *res)
{
    if (!ctx || !res || n < 2 || n_bins_half < 1 || !(eb_abs > 0.0)) return 12;
    if (!isfinite(2.0 * eb_abs)) return 11;
    if (n_bins_half > (1u << 30)) return 12;
    // the same one-round-trip path as lc_compress_auto_f64 in absolute mode: the
    // range pass supplies the non-finite check, the anchor decision and the
    // chain-value bound the quantizer's certification uses
    lc_bounds b;
    return lc_compress_auto_f64(ctx, x, n, x_on_device, 0, eb_abs, n_bins_half, record_traces, res, &b);
}

static int lc_compress_auto_impl(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device, int eb_relative,
                                 double eb_param, uint32_t n_bins_half, int record_traces, lc_result *res,
                                 lc_bounds *bounds, const LcRangePart *range_dev)
{
    if (!ctx || !res || !bounds || n < 2 || n_bins_half < 1 || !(eb_param > 0.0) || !isfinite(eb_param)) return 12;
    if (n_bins_half > (1u << 30)) return 12;
    LcDeviceGuard guard(ctx->device);
    if (!guard.ok) LC_CUDA_OK(cudaSetDevice(ctx->device));
    LC_CUDA_OK(cudaEventRecord(ctx->ev0, ctx->stream));
    LC_CUDA_OK(cudaEventRecord(ctx->pev[0], ctx->stream));
    int rc;
    const double *dx = lc_device_input(ctx, x, n, x_on_device, &rc);
    if (rc) return rc;
    // range pass and device-side bounds: no host round trip before the quantizer
    int nb = (int)((n + 255) / 256);
    if (nb > 4 * ctx->sm_count) nb = 4 * ctx->sm_count;
    LC_CUDA_OK(lc_reserve(ctx->range_parts, sizeof(LcRangePart) * (nb + 1) + 16 + sizeof(LcQuantDyn) + 64));
    LcRangePart *parts = (LcRangePart *)ctx->range_parts.p;
    unsigned *done = (unsigned *)(parts + nb + 1);
    LcQuantDyn *dyn = (LcQuantDyn *)(((uintptr_t)(done + 4) + 63) & ~(uintptr_t)63);
    if (!range_dev) {
        LC_CUDA_OK(cudaMemsetAsync(done, 0, sizeof(unsigned), ctx->stream));
        lc_range_kernel<<<nb, 256, 0, ctx->stream>>>(dx, n, parts, done);
        ctx->launches += 1;
    }
    // the producer's fused range (lc_compress_ranged_f64) replaces the range pass
    lc_quant_setup_kernel<<<1, 32, 0, ctx->stream>>>(range_dev ? range_dev : parts + nb, dx, n, eb_relative,
                                                     eb_param, n_bins_half, dyn);
    ctx->launches += 1;
    { int _rc = lc_debug_check(ctx, "lc_quant_setup_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    ctx->rng_ptr = nullptr;
    LcQuantDyn *hdyn = (LcQuantDyn *)((char *)ctx->pinned + 512);
    if (2ull * n_bins_half <= 65536ull) rc = lc_compress_t<uint16_t>(ctx, dx, n, 0.0, n_bins_half, record_traces, res, dyn, hdyn);
    else rc = lc_compress_t<uint32_t>(ctx, dx, n, 0.0, n_bins_half, record_traces, res, dyn, hdyn);
    bounds->vmin = hdyn->vmin;
    bounds->vmax = hdyn->vmax;
    bounds->value_range = hdyn->value_range;
    bounds->eb_abs = hdyn->eb_abs;
    bounds->first_value = hdyn->first_value;
    bounds->nonfinite = hdyn->nonfinite;
    bounds->status = hdyn->status;
    return rc;
}

int lc_compress_auto_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device, int eb_relative,
                         double eb_param, uint32_t n_bins_half, int record_traces, lc_result *res, lc_bounds *bounds)
{
    return lc_compress_auto_impl(ctx, x, n, x_on_device, eb_relative, eb_param, n_bins_half, record_traces, res,
                                 bounds, nullptr);
}

int lc_compress_ranged_f64(lc_ctx *ctx, const double *x, uint64_t n, int eb_relative, double eb_param,
                           uint32_t n_bins_half, int record_traces, const void *range_dev, lc_result *res,
                           lc_bounds *bounds)
{
    if (!range_dev) return 12;
    return lc_compress_auto_impl(ctx, x, n, 1, eb_relative, eb_param, n_bins_half, record_traces, res, bounds,
                                 (const LcRangePart *)range_dev);
}

int lc_result_fetch(lc_ctx *ctx, uint8_t *code_lengths, uint8_t *payload, uint64_t *esc_idx, double *esc_val,
                    double *pe, double *pe_rec)
{
    if (!ctx) return 12;
    LcDeviceGuard guard(ctx->device);
    cudaStream_t st = ctx->stream;
    if (code_lengths) LC_CUDA_OK(cudaMemcpyAsync(code_lengths, ctx->lengths.p, ctx->nbins, cudaMemcpyDeviceToHost, st));
    const uint64_t pbytes = (ctx->cb.total_bits + 7) / 8;
    if (payload && pbytes) LC_CUDA_OK(cudaMemcpyAsync(payload, ctx->payload.p, pbytes, cudaMemcpyDeviceToHost, st));
    if (esc_idx && ctx->cb.n_esc)
        LC_CUDA_OK(cudaMemcpyAsync(esc_idx, ctx->esc_idx.p, ctx->cb.n_esc * 8, cudaMemcpyDeviceToHost, st));
    if (esc_val && ctx->cb.n_esc)
        LC_CUDA_OK(cudaMemcpyAsync(esc_val, ctx->esc_val.p, ctx->cb.n_esc * 8, cudaMemcpyDeviceToHost, st));
    if (ctx->record && pe) LC_CUDA_OK(cudaMemcpyAsync(pe, ctx->pe.p, (ctx->n - 1) * 8, cudaMemcpyDeviceToHost, st));
    if (ctx->record && pe_rec)
        LC_CUDA_OK(cudaMemcpyAsync(pe_rec, ctx->pe_rec.p, (ctx->n - 1) * 8, cudaMemcpyDeviceToHost, st));
    LC_CUDA_OK(cudaStreamSynchronize(st));
    return 0;
}

int lc_result_device(lc_ctx *ctx, const uint8_t **payload, const uint8_t **code_lengths,
                     const uint64_t **esc_idx, const double **esc_val)
{
    if (!ctx) return 12;
    if (payload) *payload = (const uint8_t *)ctx->payload.p;
    if (code_lengths) *code_lengths = (const uint8_t *)ctx->lengths.p;
    if (esc_idx) *esc_idx = (const uint64_t *)ctx->esc_idx.p;
    if (esc_val) *esc_val = (const double *)ctx->esc_val.p;
    return 0;
}

// LC_TRACE=1 diagnostics: "name host_us gpu_us" per mark since the last read
// (times relative to the first mark); clears the trace.  Returns bytes written.
int lc_trace_read(lc_ctx *ctx, char *out, int cap)
{
    if (!ctx || !out || cap <= 0) return 0;
    LcDeviceGuard guard(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    int w = 0;
    out[0] = 0;
    for (int i = 0; i < ctx->tn && w < cap - 96; ++i) {
        float ms = 0.0f;
        if (i > 0) cudaEventElapsedTime(&ms, ctx->tev[0], ctx->tev[i]);
        w += snprintf(out + w, cap - w, "%s %.1f %.1f\n", ctx->tname[i], ctx->thost[i] - ctx->thost[0], 1e3 * ms);
    }
    ctx->tn = 0;
    return w;
}

int lc_trace_mark_api(lc_ctx *ctx, const char *what)
{
    if (!ctx) return 12;
    lc_trace_mark(ctx, what);
    return 0;
}

int lc_phase_ms(lc_ctx *ctx, double *ms, int cap)
{
    if (!ctx) return 0;
    int k = 0;
    auto el = [&](int a, int b) {
        float f = -1.0f;
        if (cudaEventElapsedTime(&f, ctx->pev[a], ctx->pev[b]) != cudaSuccess) f = -1.0f;
        return (double)f;
    };
    if (ctx->last_kind == 1) {
        const int pairs[4][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}};
        for (int i = 0; i < 4 && k < cap; ++i) ms[k++] = el(pairs[i][0], pairs[i][1]);
    } else if (ctx->last_kind == 2) {
        for (int i = 0; i < 4 && k < cap; ++i) ms[k++] = -1.0;
        const int pairs[4][2] = {{5, 8}, {8, 9}, {9, 6}, {6, 7}};
        for (int i = 0; i < 4 && k < cap; ++i) ms[k++] = el(pairs[i][0], pairs[i][1]);
    }
    return k;
}

uint64_t lc_launch_count(lc_ctx *ctx) { return ctx ? ctx->launches : 0; }

int lc_ctx_set_option(lc_ctx *ctx, int key, long long value)
{
    if (!ctx || key < 0 || key >= 8) return 12;
    ctx->opt[key] = value;
    return 0;
}

long long lc_ctx_get_stat(lc_ctx *ctx, int key)
{
    if (!ctx) return -1;
    switch (key) {
    case LC_STAT_QUANT_RELAUNCHES: return ctx->quant_relaunches;
    case LC_STAT_QUANT_SERIAL: return ctx->quant_serial;
    case LC_STAT_REC_RELAUNCHES: return ctx->dec_state[31];
    case LC_STAT_REC_SERIAL: return ctx->dec_state[30];
    case LC_STAT_QUANT_EXACT_CHUNKS: return (long long)ctx->quant_exact_chunks;
    default: return -1;
    }
}

int lc_decompress_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const uint8_t *code_lengths,
                      uint64_t n_lengths, const uint8_t *payload, uint64_t payload_bytes, uint64_t payload_bits,
                      const uint64_t *esc_idx, const double *esc_val, uint64_t n_esc, int inputs_on_device,
                      double *out, int out_on_device, int64_t *esc_used)
{
    if (!ctx) return 12;
    LcDeviceGuard guard(ctx->device);
    if (!guard.ok) LC_CUDA_OK(cudaSetDevice(ctx->device));
    return lc_decompress_impl2(ctx, n, eb_abs, first_value, code_lengths, n_lengths, payload, payload_bytes,
                               payload_bits, esc_idx, esc_val, n_esc, inputs_on_device, out, out_on_device,
                               esc_used, nullptr, 0);
}

int lc_result_sync_v3(lc_ctx *ctx, uint64_t *offsets, double *starts, uint64_t *escapes, uint64_t cap,
                      uint64_t *count)
{
    if (!ctx) return 12;
    LcDeviceGuard guard(ctx->device);
    if (count) *count = ctx->nsync;
    const uint64_t k = cap < ctx->nsync ? cap : ctx->nsync;
    const uint64_t stride = ctx->nsync + 1;
    if (k) {
        if (offsets) LC_CUDA_OK(cudaMemcpyAsync(offsets, ctx->sync.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (starts)
            LC_CUDA_OK(cudaMemcpyAsync(starts, (uint64_t *)ctx->sync.p + stride, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (escapes)
            LC_CUDA_OK(cudaMemcpyAsync(escapes, (uint64_t *)ctx->sync.p + 2 * stride, k * 8, cudaMemcpyDeviceToHost,
                                       ctx->stream));
        LC_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    }
    return 0;
}

int lc_result_sync_device(lc_ctx *ctx, const uint64_t **offsets, const double **starts, const uint64_t **escapes)
{
    if (!ctx) return 12;
    const uint64_t stride = ctx->nsync + 1;
    if (offsets) *offsets = (const uint64_t *)ctx->sync.p;
    if (starts) *starts = (const double *)((const uint64_t *)ctx->sync.p + stride);
    if (escapes) *escapes = (const uint64_t *)ctx->sync.p + 2 * stride;
    return 0;
}

int lc_decompress_v3_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const uint8_t *code_lengths,
                         uint64_t n_lengths, const uint8_t *payload, uint64_t payload_bytes, uint64_t payload_bits,
                         const uint64_t *sync, const double *sync_starts, const uint64_t *sync_esc, uint64_t n_sync,
                         uint32_t sync_k, const uint64_t *esc_idx, const double *esc_val, uint64_t n_esc,
                         int inputs_on_device, double *out, int out_on_device, int64_t *esc_used)
{
    if (!ctx) return 12;
    if (!sync || !sync_starts || !sync_esc || sync_k != LC_SYNC_K || n < 2 ||
        n_sync != (n - 1 + LC_SYNC_K - 1) / LC_SYNC_K)
        return 12;
    LcDeviceGuard guard(ctx->device);
    if (!guard.ok) LC_CUDA_OK(cudaSetDevice(ctx->device));
    return lc_decompress_impl2(ctx, n, eb_abs, first_value, code_lengths, n_lengths, payload, payload_bytes,
                               payload_bits, esc_idx, esc_val, n_esc, inputs_on_device, out, out_on_device,
                               esc_used, sync, n_sync, sync_starts, sync_esc);
}

int lc_result_sync(lc_ctx *ctx, uint64_t *offsets, uint64_t cap, uint64_t *count)
{
    if (!ctx) return 12;
    LcDeviceGuard guard(ctx->device);
    if (count) *count = ctx->nsync;
    if (offsets && cap) {
        const uint64_t k = cap < ctx->nsync ? cap : ctx->nsync;
        LC_CUDA_OK(cudaMemcpyAsync(offsets, ctx->sync.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
        LC_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    }
    return 0;
}

int lc_decompress_v2_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const uint8_t *code_lengths,
                         uint64_t n_lengths, const uint8_t *payload, uint64_t payload_bytes, uint64_t payload_bits,
                         const uint64_t *sync, uint64_t n_sync, uint32_t sync_k, const uint64_t *esc_idx,
                         const double *esc_val, uint64_t n_esc, int inputs_on_device, double *out,
                         int out_on_device, int64_t *esc_used)
{
    if (!ctx) return 12;
    if (!sync || sync_k != LC_SYNC_K || n < 2 || n_sync != (n - 1 + LC_SYNC_K - 1) / LC_SYNC_K) return 12;
    LcDeviceGuard guard(ctx->device);
    if (!guard.ok) LC_CUDA_OK(cudaSetDevice(ctx->device));
    return lc_decompress_impl2(ctx, n, eb_abs, first_value, code_lengths, n_lengths, payload, payload_bytes,
                               payload_bits, esc_idx, esc_val, n_esc, inputs_on_device, out, out_on_device,
                               esc_used, sync, n_sync);
}

// Debug/test hook: the device codebook (lc_codebook_kernel: the
// huffman.code_lengths + canonical_codes replacement) on a caller-given
// histogram, so adversarial frequency tables (ties, Fibonacci depths) can be
// checked against the reference without crafting data that produces them.
int lc_debug_codebook(lc_ctx *ctx, const uint32_t *hist, uint32_t nbins, uint8_t *lengths_out,
                      uint64_t *codes_out, int *max_len_out)
{
    if (!ctx || !hist || nbins < 1) return 12;
    LcDeviceGuard guard(ctx->device);
    cudaStream_t st = ctx->stream;
    LC_CUDA_OK(lc_reserve(ctx->hist, nbins * sizeof(uint32_t)));
    LC_CUDA_OK(lc_reserve(ctx->lengths, nbins));
    LC_CUDA_OK(lc_reserve(ctx->cw, nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->gkeys, 3 * (size_t)nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->ifreq, (size_t)nbins * sizeof(unsigned long long)));
    LC_CUDA_OK(lc_reserve(ctx->parent, 2 * (size_t)nbins * sizeof(int)));
    LC_CUDA_OK(lc_reserve(ctx->cbout, sizeof(LcCodebookOut)));
    LC_CUDA_OK(cudaMemcpyAsync(ctx->hist.p, hist, nbins * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    lc_codebook_kernel<<<1, 1024, lc_codebook_smem_bytes(), st>>>(
        (const uint32_t *)ctx->hist.p, nbins, (uint8_t *)ctx->lengths.p, (unsigned long long *)ctx->cw.p,
        (unsigned long long *)ctx->gkeys.p, (unsigned long long *)ctx->ifreq.p, (int *)ctx->parent.p,
        (LcCodebookOut *)ctx->cbout.p, nullptr, nullptr, nullptr);
    ctx->launches += 1;
    { int _rc = lc_debug_check(ctx, "lc_codebook_kernel", __FILE__, __LINE__); if (_rc) return _rc; }
    LcCodebookOut *h = (LcCodebookOut *)((char *)ctx->pinned + 1024);
    LC_CUDA_OK(cudaMemcpyAsync(h, ctx->cbout.p, sizeof(LcCodebookOut), cudaMemcpyDeviceToHost, st));
    if (lengths_out) LC_CUDA_OK(cudaMemcpyAsync(lengths_out, ctx->lengths.p, nbins, cudaMemcpyDeviceToHost, st));
    if (codes_out) LC_CUDA_OK(cudaMemcpyAsync(codes_out, ctx->cw.p, nbins * 8, cudaMemcpyDeviceToHost, st));
    LC_CUDA_OK(cudaStreamSynchronize(st));
    if (max_len_out) *max_len_out = h->max_len;
    return h->status;
}

// Debug/test hook: copy an intermediate of the last compress to host.
// what: 0 codes, 1 histogram (u32), 2 code lengths (u8), 3 codewords (u64), 5 codebook summary,
// 6 warp-tile aggregates (OffMap[ntiles + 1], then offsets / slacks / guesses)
int lc_debug_copy(lc_ctx *ctx, int what, void *host, uint64_t bytes)
{
    LcDeviceGuard guard(ctx->device);
    const void *src = what == 0 ? ctx->codes.p : what == 1 ? ctx->hist.p : what == 2 ? ctx->lengths.p
                    : what == 3 ? ctx->cw.p : what == 5 ? ctx->cbout.p : what == 6 ? ctx->tiles.p : ctx->timeline.p;
    LC_CUDA_OK(cudaMemcpyAsync(host, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LC_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return 0;
}

}  // extern "C"

cudaEvent_t lc_ev(lc_ctx *ctx, int which) { return which ? ctx->ev1 : ctx->ev0; }
