"""Device plumbing: torch supplies CUDA memory and the current stream; the
kernels themselves live in libqxcorr_b200.so (see _native.py)."""

from __future__ import annotations

import numpy as np

from . import _native as N


_TORCH = None


def torch():
    """The torch module once a CUDA device is confirmed (checked on first use;
    there is no CPU fallback)."""
    global _TORCH
    if _TORCH is None:
        import torch as _t

        if not _t.cuda.is_available():
            raise RuntimeError("paper_2509_19974_b200 needs a CUDA device (no CPU fallback)")
        _TORCH = _t
    return _TORCH


def as_device(a, dtype=None):
    """numpy array / torch tensor -> contiguous CUDA tensor (no copy if already one)."""
    t = torch()
    if isinstance(a, t.Tensor):
        x = a
        if dtype is not None and x.dtype != dtype:
            x = x.to(dtype)
        if not x.is_cuda:
            x = x.to("cuda", non_blocking=False)
        # keep row-contiguous views as they are: overlapping (sliding-window)
        # or repeated (stride-0) rows are legal read-only inputs
        if x.dim() == 2 and (x.stride(1) == 1 or x.shape[1] == 1):
            return x
        return x.contiguous()
    arr = np.ascontiguousarray(a)
    # read-only buffers, and negative strides that ascontiguousarray keeps
    # on single-element views, cannot be wrapped by torch
    if not arr.flags.writeable or any(st < 0 for st in arr.strides):
        arr = arr.copy()
    x = t.from_numpy(arr)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.to("cuda").contiguous()


def stream_handle() -> int:
    """Raw handle of the current CUDA stream of the current device (the
    kernels are enqueued there)."""
    t = torch()
    return t._C._cuda_getCurrentRawStream(t.cuda.current_device())


DTYPE_CODE = {"float32": N.QX_F32, "float64": N.QX_F64, "int64": N.QX_I64}


def dtype_code(x) -> int:
    name = str(x.dtype).replace("torch.", "")
    try:
        return DTYPE_CODE[name]
    except KeyError:
        raise ValueError(f"unsupported sample dtype {x.dtype} (float32, float64 or int64)") from None


def signals(x, start: int = 0) -> N.QxSignals:
    """QxSignals descriptor of a CUDA tensor shaped (n,) or (batch, n)."""
    if x.dim() == 1:
        n, ld = x.shape[0], x.shape[0]
    elif x.dim() == 2:
        # a size-1 dimension may carry any stride in torch; rows are what matter
        n = x.shape[1]
        ld = x.stride(0) if x.shape[0] > 1 else n
        if x.stride(1) != 1 and n > 1:
            raise ValueError("rows must be contiguous")
    else:
        raise ValueError("signals must be 1-D or (batch, n)")
    return N.QxSignals(x.data_ptr(), dtype_code(x), 0, int(n), int(ld), int(start))
