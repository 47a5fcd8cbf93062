"""ctypes binding of the sm_100a codec library (include/lossyckpt_b200.h).

The library is built in-tree by paper_1805_07384_b200.build (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "liblossyckpt_b200.so")

STATUS_INTEGRITY = {1: "Huffman decode failed: invalid codeword",
                    2: "Huffman decode failed: payload exhausted mid-symbol",
                    3: "Huffman decode failed: trailing bits after last symbol",
                    5: "escape positions disagree with escape codes",
                    6: "sync table disagrees with the payload"}
STATUS_PARAMETER = {10: "input contains NaN or Inf",
                    11: "error bound too large to quantize",
                    12: "invalid argument",
                    13: "code length exceeds 64 bits"}


class LcResult(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("payload_bits", ctypes.c_uint64),
                ("payload_bytes", ctypes.c_uint64), ("n_esc", ctypes.c_uint64),
                ("n_symbols", ctypes.c_uint32), ("max_len", ctypes.c_uint32),
                ("used_symbols", ctypes.c_uint32), ("relaunches", ctypes.c_uint32)]


class LcBounds(ctypes.Structure):
    _fields_ = [("vmin", ctypes.c_double), ("vmax", ctypes.c_double), ("value_range", ctypes.c_double),
                ("eb_abs", ctypes.c_double), ("first_value", ctypes.c_double), ("nonfinite", ctypes.c_int),
                ("status", ctypes.c_int)]


STATUS_CONSTANT = 15        # lc_compress_auto_f64: constant vector (reference constant block)


class LcStats(ctypes.Structure):
    _fields_ = [("sum_sq_err", ctypes.c_double), ("max_abs_err", ctypes.c_double),
                ("vmin", ctypes.c_double), ("vmax", ctypes.c_double),
                ("max_identity_dev", ctypes.c_double), ("nonfinite", ctypes.c_int),
                ("pad", ctypes.c_int)]


_vp = ctypes.c_void_p
_lib = None
_lib_lock = threading.Lock()


def library():
    """Load (never silently skip) the native codec library."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native codec library missing: {LIB_PATH} "
                               "(run python -m paper_1805_07384_b200.build)")
        L = ctypes.CDLL(LIB_PATH)
        L.lc_ctx_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _vp]
        L.lc_ctx_create.restype = ctypes.c_int
        L.lc_ctx_destroy.argtypes = [_vp]
        L.lc_ctx_destroy.restype = None
        L.lc_last_error.argtypes = [_vp]
        L.lc_last_error.restype = ctypes.c_char_p
        L.lc_range_f64.argtypes = [_vp, _vp, ctypes.c_uint64, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int)]
        L.lc_range_f64.restype = ctypes.c_int
        L.lc_compress_f64.argtypes = [_vp, _vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(LcResult)]
        L.lc_compress_f64.restype = ctypes.c_int
        L.lc_compress_auto_f64.argtypes = [_vp, _vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                           ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(LcResult),
                                           ctypes.POINTER(LcBounds)]
        L.lc_compress_auto_f64.restype = ctypes.c_int
        L.lc_result_fetch.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.lc_result_fetch.restype = ctypes.c_int
        L.lc_result_device.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                       ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
        L.lc_result_device.restype = ctypes.c_int
        L.lc_decompress_f64.argtypes = [_vp, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                        _vp, ctypes.c_uint64, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                        _vp, _vp, ctypes.c_uint64, ctypes.c_int, _vp, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int64)]
        L.lc_decompress_f64.restype = ctypes.c_int
        L.lc_last_device_ms.argtypes = [_vp]
        L.lc_last_device_ms.restype = ctypes.c_double
        L.lc_phase_ms.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.lc_phase_ms.restype = ctypes.c_int
        L.lc_launch_count.argtypes = [_vp]
        L.lc_launch_count.restype = ctypes.c_uint64
        L.lc_trace_mark_api.argtypes = [_vp, ctypes.c_char_p]
        L.lc_trace_mark_api.restype = ctypes.c_int
        L.lc_trace_read.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int]
        L.lc_trace_read.restype = ctypes.c_int
        L.lc_error_stats_f64.argtypes = [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_int, _vp, _vp,
                                         ctypes.POINTER(LcStats)]
        L.lc_error_stats_f64.restype = ctypes.c_int
        _d = ctypes.c_double
        _dp = ctypes.POINTER(ctypes.c_double)
        L.lc_stencil_apply_f64.argtypes = [_vp, _vp, _vp, _vp]
        L.lc_residual_f64.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _dp]
        L.lc_jacobi_step_f64.argtypes = [_vp, _vp, _d, _vp, _vp, _vp, _vp, _vp, _vp, _dp]
        L.lc_dot_f64.argtypes = [_vp, _vp, _vp, ctypes.c_uint64, _vp, _dp]
        L.lc_axpy_f64.argtypes = [_vp, _d, _vp, _d, _vp, _vp, ctypes.c_uint64]
        for f in (L.lc_stencil_apply_f64, L.lc_residual_f64, L.lc_jacobi_step_f64, L.lc_dot_f64, L.lc_axpy_f64):
            f.restype = ctypes.c_int
        _u64 = ctypes.c_uint64
        L.lc_result_sync_v3.argtypes = [_vp, _vp, _vp, _vp, _u64, ctypes.POINTER(ctypes.c_uint64)]
        L.lc_result_sync_v3.restype = ctypes.c_int
        L.lc_decompress_v3_f64.argtypes = [_vp, _u64, _d, _d, _vp, _u64, _vp, _u64, _u64, _vp, _vp, _vp, _u64,
                                           ctypes.c_uint32, _vp, _vp, _u64, ctypes.c_int, _vp, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int64)]
        L.lc_decompress_v3_f64.restype = ctypes.c_int
        L.lc_result_sync_device.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
        L.lc_result_sync_device.restype = ctypes.c_int
        L.lc_compress_ranged_f64.argtypes = [_vp, _vp, _u64, ctypes.c_int, _d, ctypes.c_uint32, ctypes.c_int, _vp,
                                             ctypes.POINTER(LcResult), ctypes.POINTER(LcBounds)]
        L.lc_kr_spmv_f64.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.lc_kr_residual_f64.argtypes = [_vp, _vp, _vp, _vp, _vp, _d, _vp, _vp, _vp]
        L.lc_kr_cg_update_f64.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp, _d, _vp, _vp, _vp]
        L.lc_kr_cg_dir_f64.argtypes = [_vp, _u64, _vp, _vp, _d, _vp]
        L.lc_kr_jacobi_f64.argtypes = [_vp, _vp, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.lc_kr_dot_f64.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp]
        L.lc_kr_subh_f64.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp]
        L.lc_kr_div_f64.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp]
        L.lc_kr_combine_f64.argtypes = [_vp, _u64, ctypes.c_int, _vp, _u64, _vp, _vp, _vp, _vp]
        L.lc_kr_fold_f64.argtypes = [_vp, _vp, ctypes.c_int, _u64, ctypes.c_int, _vp, _vp, _vp, _u64, _vp]
        for f in KRYLOV:
            getattr(L, f).restype = ctypes.c_int
        L.lc_compress_ranged_f64.restype = ctypes.c_int
        L.lc_ctx_set_option.argtypes = [_vp, ctypes.c_int, ctypes.c_longlong]
        L.lc_ctx_set_option.restype = ctypes.c_int
        L.lc_ctx_get_stat.argtypes = [_vp, ctypes.c_int]
        L.lc_ctx_get_stat.restype = ctypes.c_longlong
        L.lc_debug_codebook.argtypes = [_vp, _vp, ctypes.c_uint32, _vp, _vp, ctypes.POINTER(ctypes.c_int)]
        L.lc_debug_codebook.restype = ctypes.c_int
        L.lc_result_sync.argtypes = [_vp, _vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        L.lc_result_sync.restype = ctypes.c_int
        L.lc_decompress_v2_f64.argtypes = [_vp, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _vp,
                                           ctypes.c_uint64, _vp, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                           ctypes.c_uint64, ctypes.c_uint32, _vp, _vp, ctypes.c_uint64,
                                           ctypes.c_int, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
        L.lc_decompress_v2_f64.restype = ctypes.c_int
        _lib = L
        return L


EXPORTED = ["lc_ctx_create", "lc_ctx_destroy", "lc_last_error", "lc_range_f64", "lc_compress_f64",
            "lc_result_fetch", "lc_result_device", "lc_decompress_f64", "lc_last_device_ms",
            "lc_phase_ms", "lc_launch_count", "lc_error_stats_f64", "lc_stencil_apply_f64",
            "lc_residual_f64", "lc_jacobi_step_f64", "lc_dot_f64", "lc_axpy_f64", "lc_result_sync",
            "lc_decompress_v2_f64", "lc_trace_mark_api", "lc_trace_read", "lc_compress_auto_f64", "lc_ctx_set_option", "lc_ctx_get_stat",
            "lc_debug_codebook", "lc_compress_ranged_f64", "lc_result_sync_v3", "lc_decompress_v3_f64",
            "lc_result_sync_device"]
KRYLOV = ["lc_kr_spmv_f64", "lc_kr_residual_f64", "lc_kr_cg_update_f64", "lc_kr_cg_dir_f64", "lc_kr_jacobi_f64",
          "lc_kr_dot_f64", "lc_kr_subh_f64", "lc_kr_div_f64", "lc_kr_combine_f64", "lc_kr_fold_f64"]
EXPORTED = EXPORTED + KRYLOV


class Context:
    """One codec context (CUDA stream + scratch) per device and host thread."""

    def __init__(self, device=0, stream=None):
        self.lib = library()
        self.h = _vp()
        rc = self.lib.lc_ctx_create(ctypes.byref(self.h), int(device), stream)
        if rc != 0:
            raise RuntimeError(f"lc_ctx_create failed ({rc}): CUDA device {device} unavailable")
        self.device = device

    def error(self):
        return self.lib.lc_last_error(self.h).decode()

    def close(self):
        if self.h:
            self.lib.lc_ctx_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx_local = threading.local()
_MAX_STREAM_CTXS = 8          # cached contexts per thread (one per (device, stream) pair)


def _ctx_map():
    ctxs = getattr(_ctx_local, "ctxs", None)
    if ctxs is None:
        ctxs = _ctx_local.ctxs = {}
    return ctxs


def _for_stream(device, stream_ptr):
    ctxs = _ctx_map()
    key = (int(device), int(stream_ptr))
    ctx = ctxs.pop(key, None)
    if ctx is None:
        ctx = Context(device, stream=_vp(stream_ptr) if stream_ptr else None)
        ctx.stream = int(stream_ptr)
        while len(ctxs) >= _MAX_STREAM_CTXS:       # evict the least recently used
            ctxs.pop(next(iter(ctxs))).close()
    ctxs[key] = ctx                               # most recently used last
    return ctx


def bind_stream(device, stream_ptr):
    """Context for `device` whose launches go to the given CUDA stream
    (cudaStream_t as int).  Kept for callers that pass a raw stream; `context`
    already follows torch's current stream."""
    return _for_stream(device, stream_ptr)


def context(device=0):
    """This thread's codec context for `device`, ordered on torch's current CUDA
    stream of that device: the codec's kernels start after the work already
    queued on that stream (e.g. the kernel that produced x) and later work on it
    sees the codec's outputs, whatever stream the caller made current."""
    import torch
    stream = torch.cuda.current_stream(int(device)).cuda_stream
    return _for_stream(device, stream)
