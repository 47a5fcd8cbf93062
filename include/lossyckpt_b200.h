/*
 * lossyckpt_b200.h -- C ABI of the B200 (sm_100a) lossy-checkpoint codec.
 *
 * Drop-in replacement for the compute core of the reference package
 * lossyckpt (Python + numba, /root/reference/pkg/src/lossyckpt).  Plain
 * pointers and sizes only; no torch types.  The Python host layer
 * (paper_1805_07384_b200/compressor.py) binds these with ctypes exactly where
 * the reference calls its numba kernels; INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Reference interfaces replaced (file:line under pkg/src/lossyckpt/):
 *   lc_range_f64        np.isfinite / max / min        compressor.py:384-386
 *   lc_compress_f64     _compress_kernel + bincount +
 *                       huffman.code_lengths + encode  compressor.py:400-413,
 *                                                      huffman.py:21-55,96-107,135-150
 *   lc_result_fetch     the CompressedBlock fields     compressor.py:414-417
 *   lc_decompress_f64   huffman.decode + _decompress_kernel + checks
 *                                                      compressor.py:430-439,
 *                                                      huffman.py:110-132,153-172
 *   lc_error_stats_f64  measured_psnr reductions + error_identity_check
 *                                                      compressor.py:81-94,443-460
 *   lc_stencil_apply_f64, lc_residual_f64, lc_jacobi_step_f64, lc_dot_f64,
 *   lc_axpy_f64         solver harness: spmv / residual / Jacobi step /
 *                       dot / axpy of solvers.py:92-241, sparse.py:150-157
 *
 * Status codes (return values):
 *   0 ok
 *   1 invalid codeword           -> IntegrityError("Huffman decode failed: invalid codeword")
 *   2 payload exhausted          -> IntegrityError("... payload exhausted mid-symbol")
 *   3 trailing bits              -> IntegrityError("... trailing bits after last symbol")
 *   4 escape count mismatch      -> IntegrityError("escape count mismatch: ...")
 *   5 escape positions mismatch  -> IntegrityError("escape positions disagree with escape codes")
 *   6 v2 sync table mismatch     -> IntegrityError("sync table disagrees with the payload")
 *  10 non-finite input           -> ParameterError("input contains NaN or Inf")
 *  11 error bound overflow       -> ParameterError("error bound too large to quantize")
 *  12 bad argument               -> ParameterError
 *  13 code length > 64           -> ParameterError("code length exceeds 64 bits")
 *  20 CUDA error (message via lc_last_error)
 *
 * Threading: one context per host thread / CUDA stream.  Every call is
 * stream-ordered on the context's stream and returns after the results it
 * reports are final (one scalar readback per call, no other host syncs).
 */
#ifndef LOSSYCKPT_B200_H
#define LOSSYCKPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lc_ctx lc_ctx;

/* Create a context on `device` whose work is ordered on `stream` (a
 * cudaStream_t cast to void*; NULL = the legacy default stream).          */
int lc_ctx_create(lc_ctx **out, int device, void *stream);
void lc_ctx_destroy(lc_ctx *ctx);
const char *lc_last_error(lc_ctx *ctx);

/* compressor.py:384-386: min, max and a non-finite flag of x[0..n).       */
int lc_range_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device,
                 double *vmin, double *vmax, int *nonfinite);

typedef struct {
    uint64_t n;            /* elements */
    uint64_t payload_bits; /* huffman.encode bit length                   */
    uint64_t payload_bytes;/* ceil(payload_bits / 8)                       */
    uint64_t n_esc;        /* escapes                                      */
    uint32_t n_symbols;    /* 2 * n_bins_half (length of code_lengths)     */
    uint32_t max_len;      /* longest Huffman code                         */
    uint32_t used_symbols; /* symbols with a non-zero frequency            */
    uint32_t relaunches;   /* exact-chain repair passes (diagnostic)       */
} lc_result;

/* compressor.py:400-413 for n >= 2 and a non-constant vector: quantize with
 * the closed-loop order-1 predictor at eb_abs, histogram, build the Huffman
 * code on device and encode.  x is device or host memory.  Results stay in
 * the context until lc_result_fetch / lc_result_device.  Runs the value-range
 * pass like lc_compress_auto_f64 (absolute mode): returns 10 for non-finite
 * input and 15 for a constant vector (no results).                        */
int lc_compress_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device,
                    double eb_abs, uint32_t n_bins_half, int record_traces,
                    lc_result *res);

/* Bounds of an lc_compress_auto_f64 call, resolved on the device.         */
typedef struct {
    double vmin, vmax;     /* compressor.py:386 x.min(), x.max()           */
    double value_range;    /* vmax - vmin (+0.0 when equal)                */
    double eb_abs;         /* resolve_bounds (compressor.py:138-148)       */
    double first_value;    /* x[0]                                         */
    int nonfinite;         /* x holds NaN or Inf                           */
    int status;            /* 0, 10, 11, 12 or 15 (= the return value)     */
} lc_bounds;

/* compressor.py:381-413 in one host round trip: value range (non-finite
 * check), bounds (eb_abs = eb_param * value_range when eb_relative, else
 * eb_param), the 2*eb check and, for a non-constant vector, the whole
 * compression of lc_compress_f64 -- the quantizer reads the bounds the
 * device derived, so nothing waits for the host between the range pass and
 * the encoder.  Returns 0 with results, 10 (non-finite input), 11 (2*eb not
 * finite), 12 (bad argument / eb_abs <= 0) or 15 (constant vector: the
 * caller writes the reference's constant block from *bounds); *bounds is
 * filled whenever the passes ran.  Replaces compressor.py:381-413 (range,
 * resolve_bounds call, checks, _compress_kernel, bincount, encode).      */
int lc_compress_auto_f64(lc_ctx *ctx, const double *x, uint64_t n, int x_on_device,
                         int eb_relative, double eb_param, uint32_t n_bins_half,
                         int record_traces, lc_result *res, lc_bounds *bounds);

/* lc_compress_auto_f64 for a device vector whose value range its producer
 * already computed (range_dev: device LcRangePart {double vmin, vmax,
 * maxstep; int nonfinite} -- lc_kr_fold_f64's range_out; maxstep may be any
 * upper bound of |x_i - x_{i-1}|): the value-range pass over x is skipped, so
 * a checkpoint of solver state reads x once (compressor.py:384-387 fused
 * into the solver's update kernel).  Same results and statuses.          */
int lc_compress_ranged_f64(lc_ctx *ctx, const double *x, uint64_t n, int eb_relative, double eb_param,
                           uint32_t n_bins_half, int record_traces, const void *range_dev, lc_result *res,
                           lc_bounds *bounds);

/* Copy the last compress result to host buffers (any may be NULL):
 * code_lengths[n_symbols], payload[payload_bytes], esc_idx/esc_val[n_esc],
 * pe/pe_rec[n-1] (only when record_traces was set).                       */
int lc_result_fetch(lc_ctx *ctx, uint8_t *code_lengths, uint8_t *payload,
                    uint64_t *esc_idx, double *esc_val, double *pe, double *pe_rec);

/* Device pointers of the last compress result (valid until the next
 * compress on this context); any argument may be NULL.                    */
int lc_result_device(lc_ctx *ctx, const uint8_t **payload, const uint8_t **code_lengths,
                     const uint64_t **esc_idx, const double **esc_val);

/* compressor.py:420-440 for a non-constant block.  All inputs are host
 * pointers unless inputs_on_device; out is host or device memory.
 * *esc_used receives the escape count the codes require (-1 when they need
 * more than n_esc), matching the reference's error message.               */
int lc_decompress_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value,
                      const uint8_t *code_lengths, uint64_t n_lengths,
                      const uint8_t *payload, uint64_t payload_bytes, uint64_t payload_bits,
                      const uint64_t *esc_idx, const double *esc_val, uint64_t n_esc,
                      int inputs_on_device, double *out, int out_on_device,
                      int64_t *esc_used);

/* Wall time of the last compress / decompress call on the device (ms),
 * measured with CUDA events around the whole stream-ordered call.          */
double lc_last_device_ms(lc_ctx *ctx);

/* Per-phase device times of the last call (CUDA events on the context's
 * stream).  Compress: [0] range-independent setup, [1] quantizer (all
 * launches incl. repairs), [2] codebook, [3] encoder.  Decompress: [4]
 * Huffman tables + segment sync passes, [5] count scan, [6] symbol write +
 * status, [7] reconstruction.
 * Returns the number of phases written.                                    */
int lc_phase_ms(lc_ctx *ctx, double *ms, int cap);

/* Kernels this context has launched since creation (diagnostic count).   */
uint64_t lc_launch_count(lc_ctx *ctx);

/* Context options (tests and diagnostics; no reference counterpart):
 *   0 LC_OPT_MAX_QUANT     quantizer relaunches before the sequential exact
 *                          chain finishes the vector (default 64)
 *   1 LC_OPT_MAX_REC       the same for the decoder's reconstruction (64)
 *   2 LC_OPT_INJECT_QUANT  perturb the predicted start of this chunk on the
 *                          first launch (forces a relaunch; -1 off)
 *   3 LC_OPT_INJECT_REC    the same in the decoder (-1 off)
 *   4 LC_OPT_VERIFY        1: the quantizer re-runs every chunk with the exact
 *                          reference step and checks every chunk end (no
 *                          certified skip); 0 default
 *   5 LC_OPT_QUANT_RESUME  1 (default): a failed chunk prediction resumes the
 *                          exact pass from the failing chunk (pass A kept, new
 *                          offsets by a map scan); 0: relaunch the quantizer
 * lc_ctx_get_stat: 0 quantizer relaunches and 1 sequential-fallback flag of the
 * last compress, 2 / 3 the same for the last decompress, 4 chunks the last
 * compress re-ran exactly (uncertified).  Returns -1 for unknown keys.     */
int lc_ctx_set_option(lc_ctx *ctx, int key, long long value);
/* Test hook: run the device codebook build (the replacement of
 * huffman.code_lengths + canonical_codes, huffman.py:21-72) on a host
 * histogram of nbins u32 counts; lengths_out[nbins] / codes_out[nbins]
 * (host, optional) receive the code lengths and canonical codewords, and
 * *max_len_out the longest length.  Returns 0, or 13 for lengths > 64.    */
int lc_debug_codebook(lc_ctx *ctx, const uint32_t *hist, uint32_t nbins, uint8_t *lengths_out,
                      uint64_t *codes_out, int *max_len_out);
long long lc_ctx_get_stat(lc_ctx *ctx, int key);

/* Diagnostics by environment (read at context creation): LC_DEBUG_SYNC=1
 * synchronises and checks after every launch the library names (a CUDA
 * fault is then reported at its kernel); with LC_DEBUG_LOG=1 as well every
 * such launch is named on stderr before and after its synchronisation (a
 * hang shows the kernel that never returned).                              */
/* Launch timeline (diagnostics; contexts created with LC_TRACE=1 in the
 * environment): lc_trace_mark_api adds a named mark, every launch adds one
 * with the kernel name; lc_trace_read syncs the stream, writes one line
 * "name host_us gpu_us" per mark (host enqueue time and device completion
 * time, both relative to the first mark) and clears the trace.  Returns the
 * bytes written (0 when tracing is off).                                    */
int lc_trace_mark_api(lc_ctx *ctx, const char *what);
int lc_trace_read(lc_ctx *ctx, char *out, int cap);

/* Distortion statistics of a reconstruction in one fused pass: the sum of
 * squared errors sum((x - y)^2) (compensated; MSE = sum / n), max |x - y|,
 * min/max of x (value range), a non-finite flag and, when pe / pe_rec (the
 * n-1 compression traces) are given, the error-identity deviation
 * max(|x_0 - y_0|, max_i |(x_i - y_i) - (pe_{i-1} - pe_rec_{i-1})|)
 * (else -1).  Replaces the numpy reductions of measured_psnr
 * (compressor.py:81-94) and error_identity_check (compressor.py:443-460).  */
typedef struct lc_stats {
    double sum_sq_err;
    double max_abs_err;
    double vmin;
    double vmax;
    double max_identity_dev;
    int nonfinite;
    int pad;
} lc_stats;

int lc_error_stats_f64(lc_ctx *ctx, const double *original, const double *recon, uint64_t n,
                       int on_device, const double *pe, const double *pe_rec, lc_stats *out);

/* ---- v2 blocks ------------------------------------
 * A v2 block carries the bit offset of every LC_SYNC_K (= 1024)-th symbol, so
 * decoding needs no segment synchronisation.  Every compress records them;
 * lc_result_sync copies min(cap, count) offsets (count = ceil((n-1)/1024)).  */
int lc_result_sync(lc_ctx *ctx, uint64_t *offsets, uint64_t cap, uint64_t *count);
/* lc_decompress_f64 for a v2 block: sync[n_sync] bit offsets, sync_k = 1024. */
int lc_decompress_v2_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value,
                         const uint8_t *code_lengths, uint64_t n_lengths, const uint8_t *payload,
                         uint64_t payload_bytes, uint64_t payload_bits, const uint64_t *sync,
                         uint64_t n_sync, uint32_t sync_k, const uint64_t *esc_idx,
                         const double *esc_val, uint64_t n_esc, int inputs_on_device, double *out,
                         int out_on_device, int64_t *esc_used);

/* ---- solver harness (device pointers only) -------------------------------
 * Constant-coefficient 7-point stencil on an nx x ny x nz grid, x fastest
 * (k = (z*ny + y)*nx + x), Dirichlet: neighbours outside the grid are dropped.
 * 2-D problems use nz = 1.  Replaces spmv (sparse.py:21-28,150-157) for the
 * stencil matrices of the configs (generate_poisson2d, sparse.py:184-206);
 * rows are accumulated in CSR column order (z-1, y-1, x-1, centre, x+1,
 * y+1, z+1) with unfused multiply/add, bit-identical to the reference.
 * Reductions are deterministic for a given n.  *_dev outputs stay on the
 * device (NULL: scratch); *_host (optional) receives the value after a sync. */
typedef struct lc_stencil {
    int64_t nx, ny, nz;
    double c, xm, xp, ym, yp, zm, zp;
} lc_stencil;

/* y = A x                                                                  */
int lc_stencil_apply_f64(lc_ctx *ctx, const lc_stencil *s, const double *x, double *y);
/* r = b - A x, sumsq = sum r^2                                              */
int lc_residual_f64(lc_ctx *ctx, const lc_stencil *s, const double *x, const double *b, double *r,
                    double *sumsq_dev, double *sumsq_host);
/* one Jacobi step (solvers.py:104-110): x_out = x + inv*r, r_out = b - A x_out,
 * sumsq = sum r_out^2 (one launch + the final sum)                          */
int lc_jacobi_step_f64(lc_ctx *ctx, const lc_stencil *s, double inv_diag, const double *x, const double *r,
                       const double *b, double *x_out, double *r_out, double *sumsq_dev, double *sumsq_host);
/* dot = a . b                                                               */
int lc_dot_f64(lc_ctx *ctx, const double *a, const double *b, uint64_t n, double *dot_dev, double *dot_host);
/* y += alpha x, alpha = a_scale * (*a_dev) when a_dev is set, else a         */
int lc_axpy_f64(lc_ctx *ctx, double a, const double *a_dev, double a_scale, const double *x, double *y,
                uint64_t n);

/* ---- v3 blocks (continued) ---------------------------
 * A v3 block adds, at every LC_SYNC_K-th symbol, the exact chain value before
 * it (the reconstruction x'[1024 k]) and the number of escape codes before
 * it.  Every interval then decodes and reconstructs independently: one
 * kernel, no segment synchronisation, no offset maps (lc_dec_v3_kernel).
 * Codes, payload and escapes are the reference's; the tables only add
 * 24 bytes per 1024 symbols.  lc_result_sync_v3 copies the last compress's
 * tables (any pointer may be NULL); lc_decompress_v3_f64 decodes a v3 block
 * (status 6 when a table entry disagrees with the payload or the chain).    */
int lc_result_sync_v3(lc_ctx *ctx, uint64_t *offsets, double *starts, uint64_t *escapes, uint64_t cap,
                      uint64_t *count);
/* Device pointers of the last compress's sync tables (valid until the next
 * compress on this context); any argument may be NULL.                    */
int lc_result_sync_device(lc_ctx *ctx, const uint64_t **offsets, const double **starts, const uint64_t **escapes);
int lc_decompress_v3_f64(lc_ctx *ctx, uint64_t n, double eb_abs, double first_value, const uint8_t *code_lengths,
                         uint64_t n_lengths, const uint8_t *payload, uint64_t payload_bytes, uint64_t payload_bits,
                         const uint64_t *sync, const double *sync_starts, const uint64_t *sync_esc, uint64_t n_sync,
                         uint32_t sync_k, const uint64_t *esc_idx, const double *esc_val, uint64_t n_esc,
                         int inputs_on_device, double *out, int out_on_device, int64_t *esc_used);

/* ---- device-resident Krylov harness (lc_krylov.cu) -------------------------
 * Slab of a global stencil grid: planes [z0, z0 + nzl) of st (x fastest).
 * Vectors a stencil reads are passed as the address of their first local
 * element; the nx*ny halo planes before and after it must hold the
 * neighbouring ranks' planes wherever a neighbour exists.  Reductions are
 * sums of per-chunk partials over LC_KR_CHUNK_ELEMS consecutive GLOBAL
 * elements, folded in one fixed order (bit-identical for any slab split
 * whose slabs start on chunk boundaries).  Scalars live in lc_kscalars on
 * the device; once status != LC_KS_RUNNING the solver's kernels do nothing.
 * Replaces the per-iteration work of solvers.py:92-241 and sparse.py:150-157. */
#define LC_KR_CHUNK_ELEMS 4096
typedef struct lc_slab {
    lc_stencil st;         /* global grid and coefficients                  */
    int64_t z0, nzl;       /* first global plane, local planes             */
} lc_slab;

typedef struct lc_kscalars {
    double rho, pq, alpha, beta;
    double rr;             /* last folded sum of squares                   */
    double res;            /* residual norm (solvers.py _set_residual)     */
    double tol_abs;        /* tolerance * ||b||, set by the host           */
    double spare;
    int64_t iteration;
    int32_t status;        /* LC_KS_*                                       */
    int32_t pad;
} lc_kscalars;
#define LC_KS_RUNNING 0
#define LC_KS_CONVERGED 1
#define LC_KS_BREAKDOWN 2  /* CG zero curvature or zero rho                */
#define LC_KS_NONFINITE 3  /* residual norm not finite                     */
/* fold ops */
#define LC_KOP_DOT 0           /* *out = sum                               */
#define LC_KOP_NORM 1          /* *out = sqrt(sum)                         */
#define LC_KOP_ALPHA 2         /* CG: pq = sum, alpha = rho / pq            */
#define LC_KOP_BETA 3          /* CG: rho' = sum0, beta = rho'/rho, res = sqrt(sum1), iteration++ */
#define LC_KOP_REBUILD_INIT 4  /* CG: rho = sum0, res = sqrt(sum1), converged test */
#define LC_KOP_REBUILD_STEP 5  /* CG restart inside a step: no converged test */
#define LC_KOP_RESID 6         /* Jacobi: res = sqrt(sum) (width 2: column 1), iteration++ */
#define LC_KOP_RESID_INIT 7    /* res = sqrt(sum) (width 2: column 1), converged test */

/* y = A vh on the slab; part[c] (optional) = chunk sums of vh*y             */
int lc_kr_spmv_f64(lc_ctx *ctx, const lc_slab *s, const double *vh, double *y, double *part,
                   const lc_kscalars *sc);
/* r = b - A xh; z_p (optional) = inv*r; part[2c] = sum r*z, part[2c+1] = sum r^2 */
int lc_kr_residual_f64(lc_ctx *ctx, const lc_slab *s, const double *xh, const double *b, double *r,
                       double inv_diag, double *z_p, double *part, const lc_kscalars *sc_gate);
/* CG (solvers.py:139-143): x += alpha p, r -= alpha q, part = (r.z, r.r) per
 * chunk, range_parts (optional: one 48-byte record per chunk -- vmin, vmax,
 * max |x_k - x_{k-1}| inside the chunk, first, last, non-finite) = range of x */
int lc_kr_cg_update_f64(lc_ctx *ctx, uint64_t n, const double *p, const double *q, double *x, double *r,
                        double inv_diag, const lc_kscalars *sc, double *part, void *range_parts);
/* CG (solvers.py:145): p = inv*r + beta p                                    */
int lc_kr_cg_dir_f64(lc_ctx *ctx, uint64_t n, const double *r, double *p, double inv_diag, const lc_kscalars *sc);
/* Jacobi (solvers.py:104-110): x2 = x + inv*r, r2 = b - A x2, part = r2^2    */
int lc_kr_jacobi_f64(lc_ctx *ctx, const lc_slab *s, double inv_diag, const double *xh, const double *rh,
                     const double *b, double *x2, double *r2, const lc_kscalars *sc, double *part,
                     void *range_parts);
/* part[c] = chunk sums of a*b                                               */
int lc_kr_dot_f64(lc_ctx *ctx, uint64_t n, const double *a, const double *b, double *part, const lc_kscalars *sc);
/* y -= (*h_dev) x   (GMRES modified Gram-Schmidt, solvers.py:217-219)      */
int lc_kr_subh_f64(lc_ctx *ctx, uint64_t n, const double *x, double *y, const double *h_dev, const lc_kscalars *sc);
/* y = x / (*d_dev)  (GMRES normalisation, solvers.py:184,237)               */
int lc_kr_div_f64(lc_ctx *ctx, uint64_t n, const double *x, double *y, const double *d_dev, const lc_kscalars *sc);
/* x = xbase + sum_{i<j} y_i basis[i*ld ..]  (GMRES, solvers.py:196)         */
int lc_kr_combine_f64(lc_ctx *ctx, uint64_t n, int j, const double *basis, uint64_t ld, const double *y_dev,
                      const double *xbase, double *x, void *range_parts);
/* Fold part[nchunks][width] in the fixed order and apply op to *sc (out_dev
 * receives the DOT/NORM value, or the residual norm for the other ops);
 * range_parts (optional) fold into *range_out (vmin, vmax, maxstep = the
 * largest |x_k - x_{k-1}| including the chunk boundaries, nonfinite) for
 * lc_compress_ranged_f64 -- the same record lc_range_f64's pass produces.   */
int lc_kr_fold_f64(lc_ctx *ctx, const double *part, int width, uint64_t nchunks, int op, lc_kscalars *sc,
                   double *out_dev, const void *range_parts, uint64_t n_range_parts, void *range_out);

#ifdef __cplusplus
}
#endif
#endif
