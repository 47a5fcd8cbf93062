"""Host <-> HBM transfers for the public numpy API.

Pageable transfers run at a few GB/s (a 512 MB vector: ~50 ms in, ~110-250
ms out).  Here large host arrays move through two cached pinned buffers per
device: the DMA of one chunk overlaps the (multi-threaded) host copy of the
other, so both directions run near PCIe speed.  Device buffers owned by the
native library are viewed through __cuda_array_interface__ (no copies).

Ordering: the codec context runs on torch's current stream of the device
(_native.context), and these copies are issued on that same stream, so they
are stream-ordered after the kernels that produce their sources.  The staging
events are recorded on the stream of the device the copy runs on (not on the
current device's stream), so a buffer is reused only after its own DMA.
"""

from __future__ import annotations

import ctypes
import threading
import warnings

import numpy as np

CHUNK = 32 << 20              # bytes per pinned staging buffer
_local = threading.local()

_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]


class _DevView:
    """A raw device allocation as a torch tensor (zero copy)."""

    def __init__(self, ptr, nbytes, typestr="|u1", itemsize=1):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_bytes(ptr, nbytes, device):
    import torch
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_DevView(ptr, nbytes), device=device)


def _buffers(device):
    import torch
    key = int(device.index or 0)
    bufs = getattr(_local, "bufs", None)
    if bufs is None:
        bufs = _local.bufs = {}
    if key not in bufs:
        bufs[key] = ([torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
                     [torch.cuda.Event() for _ in range(2)])
    return bufs[key]


def to_device(host_u8, device):
    """Host uint8 tensor/array -> new device uint8 tensor (chunked, pinned)."""
    import torch
    if isinstance(host_u8, torch.Tensor):
        src = host_u8
    else:
        arr = np.ascontiguousarray(host_u8)
        with warnings.catch_warnings():          # read-only sources (bytes) are only read here
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(arr)
    src = src.reshape(-1)
    n = src.numel()
    out = torch.empty(n, dtype=torch.uint8, device=device)
    if n == 0:
        return out
    if src.is_pinned() or n <= (1 << 20):
        out.copy_(src, non_blocking=False)
        return out
    bufs, evs = _buffers(out.device)
    for i, off in enumerate(range(0, n, CHUNK)):
        k = i & 1
        m = min(CHUNK, n - off)
        evs[k].synchronize()                     # DMA that last used this buffer is done
        bufs[k][:m].copy_(src[off:off + m])
        out[off:off + m].copy_(bufs[k][:m], non_blocking=True)
        evs[k].record(torch.cuda.current_stream(out.device))
    evs[0].synchronize()
    evs[1].synchronize()
    return out


def pinned_to_device(t, chunk=CHUNK):
    """Host tensor -> new CUDA tensor on the current stream.  Large pinned sources move
    in `chunk`-byte copies so transfers of other streams (a concurrent checkpoint's
    small payload copies) are not queued behind one long DMA."""
    import torch
    if not t.is_pinned() or t.numel() * t.element_size() <= 2 * chunk:
        return t.to("cuda", non_blocking=False)
    out = torch.empty(t.shape, dtype=t.dtype, device="cuda")
    step = max(1, chunk // t.element_size())
    for off in range(0, t.numel(), step):
        out[off:off + step].copy_(t[off:off + step], non_blocking=True)
    torch.cuda.current_stream(out.device).synchronize()
    return out


def to_host_into(dev_u8, host_u8):
    """Device uint8 tensor -> existing writable host uint8 tensor (chunked, pinned)."""
    import torch
    n = dev_u8.numel()
    if n == 0:
        return
    if host_u8.is_pinned() or n <= (1 << 20):
        host_u8.copy_(dev_u8, non_blocking=False)
        return
    bufs, evs = _buffers(dev_u8.device)
    offs = list(range(0, n, CHUNK))
    for i, off in enumerate(offs + [None]):
        if off is not None:
            k = i & 1
            m = min(CHUNK, n - off)
            evs[k].synchronize()                 # host copy of this buffer finished below
            bufs[k][:m].copy_(dev_u8[off:off + m], non_blocking=True)
            evs[k].record(torch.cuda.current_stream(dev_u8.device))
        if i > 0:
            p = offs[i - 1]
            kp = (i - 1) & 1
            pm = min(CHUNK, n - p)
            evs[kp].synchronize()
            host_u8[p:p + pm].copy_(bufs[kp][:pm])


def to_numpy(dev, dtype=np.float64):
    """Device tensor -> new numpy array of `dtype`."""
    import torch
    n = dev.numel()
    out = np.empty(n, dtype=dtype)
    to_host_into(dev.reshape(-1).view(torch.uint8), torch.from_numpy(out.view(np.uint8)))
    return out


def to_bytes(dev_u8):
    """Device uint8 tensor -> new immutable bytes object (filled in place
    right after creation, before any other reference exists)."""
    import torch
    n = dev_u8.numel()
    b = _PyBytes_FromStringAndSize(None, n)
    if n:
        addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
        view = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(addr))
        to_host_into(dev_u8, torch.from_numpy(view))
    return b
