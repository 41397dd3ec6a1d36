"""torch plumbing: device placement, streams and raw pointers for the C ABI.

PyTorch only owns device memory and streams here; all compute on the path is
in libseriesearch_b200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .errors import DeviceError, UsageError


def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device is visible: this package has no CPU path")
    return t


def device_f32(a, n: int | None = None):
    """Contiguous float32 CUDA tensor view/copy of ``a`` (numpy or torch), 2-D."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        x = a
        if x.dtype != t.float32:
            x = x.float()
        if not x.is_cuda:
            x = x.pin_memory().cuda(non_blocking=True) if x.numel() > (1 << 20) else x.cuda()
    else:
        arr = np.ascontiguousarray(a, dtype=np.float32)
        x = t.from_numpy(arr).cuda()
    if x.dim() == 1:
        x = x.unsqueeze(0)
    x = x.contiguous()
    if n is not None and x.shape[-1] != n:
        raise UsageError(f"series length {x.shape[-1]} does not match {n}")
    return x


def ptr(x) -> ctypes.c_void_p:
    return ctypes.c_void_p(x.data_ptr() if x is not None else 0)


def stream_handle(stream=None) -> ctypes.c_void_p:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
