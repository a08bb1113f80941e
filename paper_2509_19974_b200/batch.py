"""Batched GPU estimation: many (x, y) pairs per call, optional lag window.

New API next to the reference's single-pair ``estimate`` (estimator.py:60-101):
``estimate_batch`` returns, per pair, the peak value, the smallest lag
attaining it and the tie count -- exactly ``int(c.values.max())``,
``argmax_set(c)[0]`` and ``len(argmax_set(c))`` of the reference correlogram
restricted to [lag_lo, lag_hi] (estimator.py:50-57, 94).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from ._call import call, raise_for
from .quantize import native_quantizer

__all__ = ["BatchResult", "EstimatePlan", "estimate_batch", "estimate_batch_host", "estimate_sweep",
           "estimate_sweep_host", "check_results", "template_search", "template_search_summary"]


@dataclass
class BatchResult:
    raw: object  # (batch, 8) int64 CUDA tensor in qx_result layout

    @property
    def value(self):
        return self.raw[:, 0]

    @property
    def lag(self):
        return self.raw[:, 1]

    @property
    def ties(self):
        return self.raw[:, 2]

    @property
    def sumsq_x(self):
        return self.raw[:, 3]

    @property
    def sumsq_y(self):
        return self.raw[:, 4]

    @property
    def flags(self):
        return self.raw[:, 7] & 0xFFFFFFFF

    @property
    def status(self):
        return self.raw[:, 7] >> 32

    def numpy(self) -> np.ndarray:
        return self.raw.cpu().numpy().view(N.RESULT_DTYPE).reshape(-1)


def _bounds(lag_lo, lag_hi):
    return (N.INT64_MIN if lag_lo is None else int(lag_lo),
            N.INT64_MAX if lag_hi is None else int(lag_hi))


def estimate_batch(x, y, qx, qy, *, lag_lo=None, lag_hi=None, x_start=0, y_start=0, path="auto",
                   out=None) -> BatchResult:
    """Peak summaries of B pairs: x (B, Nx), y (B, Ny) CUDA tensors (or
    arrays, copied to the device), float32/float64 samples (or int64 codes
    with integer bounds as qx/qy).  Enqueued on the current stream."""
    t = D.torch()
    x = D.as_device(x)
    y = D.as_device(y)
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if y.dim() == 1:
        y = y.unsqueeze(0)
    if x.shape[0] != y.shape[0]:
        raise ValueError("x and y must hold the same number of rows")
    batch = x.shape[0]
    raw = out if out is not None else t.empty((batch, 8), dtype=t.int64, device=x.device)
    nqx, kx = native_quantizer(qx)
    nqy, ky = native_quantizer(qy)
    sx, sy = D.signals(x, x_start), D.signals(y, y_start)
    lo, hi = _bounds(lag_lo, lag_hi)
    ctx = N.context(x.device.index)
    call(N.load().qx_estimate_batch, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, ctypes.byref(nqx),
         ctypes.byref(nqy), lo, hi, N.PATHS[path], raw.data_ptr(), D.stream_handle())
    return BatchResult(raw)


class EstimatePlan:
    """estimate_batch prepared once for repeated calls of one shape (the
    low-latency form for serving pair after pair, e.g. BASELINE config 1):
    validation, threshold tables, path choice and scratch layout happen at
    construction (qx_plan_create); each call passes only the row pointers to
    qx_plan_run and returns exactly what estimate_batch returns for the same
    rows.  `x` and `y` at construction give the shapes, dtypes, row stride and
    device (tensors or arrays; their data is not used)."""

    def __init__(self, x, y, qx, qy, *, lag_lo=None, lag_hi=None, x_start=0, y_start=0, path="auto"):
        t = D.torch()
        x = D.as_device(x)
        y = D.as_device(y)
        if x.dim() == 1:
            x = x.unsqueeze(0)
        if y.dim() == 1:
            y = y.unsqueeze(0)
        if x.shape[0] != y.shape[0]:
            raise ValueError("x and y must hold the same number of rows")
        self.batch = x.shape[0]
        self.device = x.device
        # what every call must match: row length, dtype, row stride
        self._chk = (x.shape[1], x.dtype, x.stride(0) if x.shape[0] > 1 else None,
                     y.shape[1], y.dtype, y.stride(0) if y.shape[0] > 1 else None)
        nqx, _ = native_quantizer(qx)
        nqy, _ = native_quantizer(qy)
        sx, sy = D.signals(x, x_start), D.signals(y, y_start)
        lo, hi = _bounds(lag_lo, lag_hi)
        self._ctx = N.context(self.device.index)
        self._lib = N.load()
        h = ctypes.c_void_p()
        call(self._lib.qx_plan_create, self._ctx, ctypes.byref(sx), ctypes.byref(sy), self.batch,
             ctypes.byref(nqx), ctypes.byref(nqy), lo, hi, N.PATHS[path], ctypes.byref(h))
        self._h = h
        self._run = self._lib.qx_plan_run
        self._run_host = self._lib.qx_plan_run_host
        self._t = t
        self.path = {v: k for k, v in N.PATHS.items() if k != "tc"}[self._lib.qx_plan_path(h)]

    def __call__(self, x, y, out=None) -> BatchResult:
        """Enqueue the estimate of rows `x`, `y` (CUDA tensors of the plan's
        shapes, dtypes and row stride) on the current stream."""
        nx, dx, lx, ny, dy, ly = self._chk
        if x.shape[-1] != nx or y.shape[-1] != ny or x.dtype != dx or y.dtype != dy or not (x.is_cuda and y.is_cuda) \
                or (lx is not None and x.stride(0) != lx) or (ly is not None and y.stride(0) != ly):
            raise ValueError("rows do not match the plan's length / dtype / row stride, or are not CUDA tensors")
        raw = out if out is not None else self._t.empty((self.batch, 8), dtype=self._t.int64, device=self.device)
        st = self._run(self._h, x.data_ptr(), y.data_ptr(), raw.data_ptr(),
                       self._t._C._cuda_getCurrentRawStream(self.device.index))
        if st != N.QX_OK:
            raise_for(st, self._lib.qx_context_last_error(self._ctx).decode() or
                      self._lib.qx_status_string(st).decode())
        return BatchResult(raw)

    def run_host(self, x: np.ndarray, y: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """The same estimate from HOST rows (numpy arrays of the plan's shapes,
        dtypes and row stride) through qx_plan_run_host: H2D into the plan's
        own device staging, the plan's launches, D2H of the results and one
        synchronisation in a single C-ABI call.  Page-locked rows (e.g. numpy
        views of pinned torch tensors) copy by asynchronous DMA.  Returns the
        structured qx_result array; raises on the first failing pair."""
        nx, dx, lx, ny, dy, ly = self._chk
        to_np = {self._t.float32: np.float32, self._t.float64: np.float64, self._t.int64: np.int64}
        if x.shape[-1] != nx or y.shape[-1] != ny or x.dtype != to_np.get(dx) or y.dtype != to_np.get(dy) \
                or not (x.flags.c_contiguous and y.flags.c_contiguous) \
                or (x.size // nx) != self.batch or (y.size // ny) != self.batch \
                or (lx is not None and lx != nx) or (ly is not None and ly != ny):
            raise ValueError("rows do not match the plan's length / dtype / batch, or are not contiguous")
        res = out if out is not None else np.zeros(self.batch, dtype=N.RESULT_DTYPE)
        st = self._run_host(self._h, x.ctypes.data, y.ctypes.data, res.ctypes.data)
        if st != N.QX_OK:
            raise_for(st, self._lib.qx_context_last_error(self._ctx).decode() or
                      self._lib.qx_status_string(st).decode())
        return res

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.qx_plan_destroy(h)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self._h = None


def estimate_sweep(x, y, quantizers, *, lag_lo=None, lag_hi=None, x_start=0, y_start=0, path="auto",
                   out=None) -> list:
    """Several quantiser pairs over one batch of DEVICE rows (a bit-depth
    sweep) through qx_estimate_sweep: one C-ABI call whose correlations run
    on concurrent compute lanes, joined back to the current stream.
    `quantizers` is a sequence of (qx, qy); returns one BatchResult per pair
    (views of one (nq, B, 8) int64 tensor)."""
    t = D.torch()
    x = D.as_device(x)
    y = D.as_device(y)
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if y.dim() == 1:
        y = y.unsqueeze(0)
    if x.shape[0] != y.shape[0]:
        raise ValueError("x and y must hold the same number of rows")
    batch, nq = x.shape[0], len(quantizers)
    if nq < 1:
        raise ValueError("need at least one quantiser pair")
    raw = out if out is not None else t.empty((nq, batch, 8), dtype=t.int64, device=x.device)
    keep = [(native_quantizer(a), native_quantizer(b)) for a, b in quantizers]
    aqx = (N.QxQuantizer * nq)(*[k[0][0] for k in keep])
    aqy = (N.QxQuantizer * nq)(*[k[1][0] for k in keep])
    sx, sy = D.signals(x, x_start), D.signals(y, y_start)
    lo, hi = _bounds(lag_lo, lag_hi)
    ctx = N.context(x.device.index)
    call(N.load().qx_estimate_sweep, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, nq, aqx, aqy, lo, hi,
         N.PATHS[path], raw.data_ptr(), D.stream_handle())
    return [BatchResult(raw[q]) for q in range(nq)]


def estimate_batch_host(x: np.ndarray, y: np.ndarray, qx, qy, *, lag_lo=None, lag_hi=None, x_start=0,
                        y_start=0, path="auto", device=None) -> np.ndarray:
    """The same from HOST arrays through qx_estimate_batch_host (H2D, kernels,
    D2H inside one synchronous C-ABI call).  Returns a structured array with
    the qx_result fields; raises on the first failing pair."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    if x.ndim == 1:
        x = x[None]
    if y.ndim == 1:
        y = y[None]
    batch = x.shape[0]
    res = np.zeros(batch, dtype=N.RESULT_DTYPE)
    codes = {np.dtype(np.float32): N.QX_F32, np.dtype(np.float64): N.QX_F64, np.dtype(np.int64): N.QX_I64}
    sx = N.QxSignals(x.ctypes.data, codes[x.dtype], 0, x.shape[1], x.shape[1], int(x_start))
    sy = N.QxSignals(y.ctypes.data, codes[y.dtype], 0, y.shape[1], y.shape[1], int(y_start))
    nqx, kx = native_quantizer(qx)
    nqy, ky = native_quantizer(qy)
    lo, hi = _bounds(lag_lo, lag_hi)
    ctx = N.context(device)
    call(N.load().qx_estimate_batch_host, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, ctypes.byref(nqx),
         ctypes.byref(nqy), lo, hi, N.PATHS[path], res.ctypes.data)
    return res


def estimate_sweep_host(x: np.ndarray, y: np.ndarray, quantizers, *, lag_lo=None, lag_hi=None, x_start=0,
                        y_start=0, path="auto", device=None) -> np.ndarray:
    """Several quantiser pairs over one batch of HOST arrays (a bit-depth
    sweep) through qx_estimate_sweep_host: the inputs cross PCIe once, in pair
    chunks overlapped with the correlation of the previous chunk.
    `quantizers` is a sequence of (qx, qy); returns results[q, b] (structured
    qx_result fields); raises on the first failing pair."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    if x.ndim == 1:
        x = x[None]
    if y.ndim == 1:
        y = y[None]
    if x.shape[0] != y.shape[0]:
        raise ValueError("x and y batch sizes differ")
    batch, nq = x.shape[0], len(quantizers)
    if nq < 1:
        raise ValueError("need at least one quantiser pair")
    res = np.zeros((nq, batch), dtype=N.RESULT_DTYPE)
    codes = {np.dtype(np.float32): N.QX_F32, np.dtype(np.float64): N.QX_F64, np.dtype(np.int64): N.QX_I64}
    sx = N.QxSignals(x.ctypes.data, codes[x.dtype], 0, x.shape[1], x.shape[1], int(x_start))
    sy = N.QxSignals(y.ctypes.data, codes[y.dtype], 0, y.shape[1], y.shape[1], int(y_start))
    keep = [(native_quantizer(a), native_quantizer(b)) for a, b in quantizers]
    aqx = (N.QxQuantizer * nq)(*[k[0][0] for k in keep])
    aqy = (N.QxQuantizer * nq)(*[k[1][0] for k in keep])
    lo, hi = _bounds(lag_lo, lag_hi)
    ctx = N.context(device)
    call(N.load().qx_estimate_sweep_host, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, nq, aqx, aqy, lo, hi,
         N.PATHS[path], res.ctypes.data)
    return res


def template_search_summary(template, stream, qx, qy, *, stream_start: int = 0, block: int | None = None,
                            path: str = "auto"):
    """The device int64[8] summary of template_search (value, smallest lag,
    ties, NaN seen, x all-zero, y all-zero in every block, a block failed,
    its status), enqueued on the current stream and not inspected (the
    multi-GPU reduction combines these before any exception is raised)."""
    t = D.torch()
    x = D.as_device(template).reshape(-1)
    y = D.as_device(stream).reshape(-1)
    if y.shape[0] - x.shape[0] + 1 < 1:
        raise ValueError("template longer than the stream")
    if block is not None and block < 1:
        raise ValueError("template too long for the block transform")
    nqx, _ = native_quantizer(qx)
    nqy, _ = native_quantizer(qy)
    sx, sy = D.signals(x, 0), D.signals(y, stream_start)
    out = t.empty(8, dtype=t.int64, device=x.device)
    ctx = N.context(x.device.index)
    call(N.load().qx_template_search, ctx, ctypes.byref(sx), ctypes.byref(sy), ctypes.byref(nqx), ctypes.byref(nqy),
         0 if block is None else int(block), N.PATHS[path], out.data_ptr(), D.stream_handle())
    return out


def template_search(template, stream, qx, qy, *, stream_start: int = 0, block: int | None = None,
                    path: str = "auto") -> tuple[int, int, int]:
    """Peak summary (value, smallest lag, ties) of estimate(x=template, y=stream)
    over the VALID lags (template fully inside the stream):
    lag in [stream_start, stream_start + len(stream) - len(template)].

    One C-ABI call (qx_template_search): the valid-lag range is cut into
    blocks of `block` lags (default: the tensor-core tile, else the largest
    one-transform NTT block); block b correlates the template (a stride-0
    row, never copied) with the stream window [b*block, b*block + block +
    len(template) - 1) and the per-block summaries are merged on the device.
    Each block's lags use only samples inside its window, so the result
    equals the reference's argmax_set summary of the full correlogram
    restricted to the valid lags (estimator.py:50-57)."""
    out = template_search_summary(template, stream, qx, qy, stream_start=stream_start, block=block, path=path)
    vmax, lmin, nties, nan, degx, degy, anybad, badst = out.cpu().tolist()
    if nan:
        raise ValueError("input contains NaN")
    if degx:
        raise_for(N.QX_DEGENERATE_QUANTIZATION, "x quantizes to all zeros")
    if degy:
        raise_for(N.QX_DEGENERATE_QUANTIZATION, "y quantizes to all zeros")
    if anybad:
        raise_for(int(badst), "template search block failed")
    return (int(vmax), int(lmin), int(nties))


def check_results(res: np.ndarray) -> None:
    """Raise the reference exception for the first failing pair."""
    bad = np.flatnonzero(res["status"] != 0)
    if bad.size:
        i = int(bad[0])
        st, fl = int(res["status"][i]), int(res["flags"][i])
        if st == N.QX_DEGENERATE_QUANTIZATION:
            side = "x" if fl & N.RF_DEGENERATE_X else "y"
            raise_for(st, f"{side} quantizes to all zeros")
        raise_for(st, f"pair {i}: status {st}")
