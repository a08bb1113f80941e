"""Monotone, zero-fixing integer quantisers, evaluated on the GPU.

Mirrors /root/reference/pkg/src/qxcorr/quantize.py: the same ``Quantizer``
(kind in {"sign", "uniform", "custom"}, validation 37-51, ``spec`` 67-73),
constructors ``sign/uniform/custom/from_spec`` (76-102) and ``apply``
(105-107).  ``Quantizer.__call__`` and ``apply`` run the qx_quantize kernel:
exact threshold compares that reproduce the reference's float64 map
(53-65) bit for bit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _native as N
from .signals import IntSignal, Signal

__all__ = ["Quantizer", "sign", "uniform", "custom", "from_spec", "apply", "random_monotone",
           "native_quantizer", "thresholds", "quantize_packed", "unpack_codes", "packed_bits"]


@dataclass(frozen=True)
class Quantizer:
    """Monotone map from reals to integers in [-k, k] with q(0) = 0."""

    kind: str
    k: int
    step: float = 1.0
    thresholds: tuple[float, ...] = field(default=())

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("level bound k must be >= 1")
        if self.kind == "uniform" and not self.step > 0:
            raise ValueError("uniform step must be > 0")
        if self.kind == "custom":
            t = np.asarray(self.thresholds, dtype=np.float64)
            if t.size != 2 * self.k:
                raise ValueError("custom quantizer needs exactly 2k thresholds")
            if not np.all(np.diff(t) > 0):
                raise ValueError("thresholds must be strictly increasing")
            if not (t[self.k - 1] <= 0.0 < t[self.k]):
                raise ValueError("level 0 must contain the input 0")
        elif self.kind not in ("sign", "uniform"):
            raise ValueError(f"unknown quantizer kind {self.kind!r}")

    def __call__(self, values) -> np.ndarray:
        """Quantise an array (or scalar) of reals to int64 levels on the GPU."""
        v = np.asarray(values, dtype=np.float64)
        codes = quantize_device(self, D.as_device(v.reshape(-1)))
        return codes.cpu().numpy().reshape(v.shape)

    def spec(self) -> str:
        if self.kind == "sign":
            return "sign"
        if self.kind == "uniform":
            return f"uniform:{self.k}:{self.step:g}"
        return f"custom[{2 * self.k} thresholds]"


def sign() -> Quantizer:
    return Quantizer(kind="sign", k=1)


def uniform(k: int, step: float) -> Quantizer:
    return Quantizer(kind="uniform", k=k, step=step)


def custom(thresholds) -> Quantizer:
    t = tuple(float(x) for x in thresholds)
    if len(t) % 2:
        raise ValueError("threshold count must be even")
    return Quantizer(kind="custom", k=len(t) // 2, thresholds=t)


def from_spec(text: str) -> Quantizer:
    """``sign`` or ``uniform:K:STEP`` (quantize.py:92-102)."""
    parts = text.strip().split(":")
    if parts == ["sign"]:
        return sign()
    if parts[0] == "uniform" and len(parts) == 3:
        try:
            return uniform(int(parts[1]), float(parts[2]))
        except ValueError as exc:
            raise ValueError(f"bad uniform quantizer spec {text!r}: {exc}") from exc
    raise ValueError(f"unknown quantizer spec {text!r} (expected 'sign' or 'uniform:K:STEP')")


def random_monotone(seed: int, k: int, levels: int | None = None, scale: float = 1.0) -> Quantizer:
    """Seeded random custom staircase for property tests (quantize.py:110-131):
    depth d (drawn in [1, k], or (levels - 1) // 2 capped to [1, k]), 2d
    strictly increasing thresholds spanning ~[-scale, scale] with 0 inside the
    middle step.  Same draws in the same order as the reference, so a seed
    gives the reference's quantiser."""
    if k < 1:
        raise ValueError("k must be >= 1")
    rng = np.random.default_rng(seed)
    d = int(rng.integers(1, k + 1)) if levels is None else max(1, min(k, (levels - 1) // 2))
    edges = np.cumsum(rng.uniform(0.05, 1.0, size=2 * d))
    edges = edges / edges[-1] * 2.0 * scale  # (this float operation order keeps the thresholds bit-identical)
    return custom(edges - rng.uniform(edges[d - 1], edges[d]))


_KIND = {"sign": N.QX_Q_SIGN, "uniform": N.QX_Q_UNIFORM, "custom": N.QX_Q_CUSTOM}


_NATIVE_CACHE: dict = {}


def native_quantizer(q):
    """(QxQuantizer, keep-alive) for this package's or the reference's Quantizer
    (cached per immutable quantiser of this package)."""
    if isinstance(q, Quantizer):
        hit = _NATIVE_CACHE.get(q)
        if hit is None:
            if len(_NATIVE_CACHE) > 4096:
                _NATIVE_CACHE.clear()
            hit = _NATIVE_CACHE[q] = _native_quantizer(q)
        return hit
    return _native_quantizer(q)


def _native_quantizer(q):
    if isinstance(q, int):  # integer codes with this bound (IntSignal)
        return N.QxQuantizer(N.QX_Q_CODES, 0, int(q), 1.0, None), None
    kind = _KIND[q.kind]
    thr = None
    ptr = None
    if q.kind == "custom":
        thr = np.ascontiguousarray(np.asarray(q.thresholds, dtype=np.float64))
        ptr = thr.ctypes.data
    return N.QxQuantizer(kind, 0, int(q.k), float(getattr(q, "step", 1.0)), ptr), thr


def thresholds(q, dtype: str = "float32") -> np.ndarray:
    """Exact decision thresholds of ``q`` for inputs of ``dtype`` (host)."""
    nq, keep = native_quantizer(q)
    return N.thresholds(nq, N.QX_F32 if dtype == "float32" else N.QX_F64, int(q.k))


def quantize_device(q, x, with_stats: bool = False):
    """int64 codes of a CUDA tensor x ((n,) or (batch, n)), float32/float64."""
    t = D.torch()
    if x.dtype not in (t.float32, t.float64):
        x = x.to(t.float64)
    batch = x.shape[0] if x.dim() == 2 else 1
    codes = t.empty(x.shape, dtype=t.int64, device=x.device)
    sums = t.zeros((2, batch), dtype=t.int64, device=x.device)
    nq, keep = native_quantizer(q)
    sig = D.signals(x)
    ctx = N.context(x.device.index)
    N.check(N.load().qx_quantize(ctx, ctypes.byref(nq), ctypes.byref(sig), batch, codes.data_ptr(),
                                 sums[0].data_ptr(), sums[1].data_ptr(), D.stream_handle()), ctx)
    del keep
    if with_stats:
        return codes, sums
    return codes


def packed_bits(q) -> int:
    """Narrowest packed field that holds every code of q (0: none does)."""
    k = int(q.k)
    return 2 if k <= 1 else 4 if k <= 7 else 8 if k <= 127 else 0


def quantize_packed(q, x, bits: int | None = None):
    """Bit-packed codes of a CUDA tensor x ((n,) or (batch, n), float32 or
    float64) through qx_quantize_packed: (codes, sumsq, nnz, flags) with codes
    a uint32 tensor (batch, qx_packed_words(n, bits)) in the layout of
    include/qxcorr_b200.h (two's-complement b-bit fields for bits = 2, 4, 8;
    sign and nonzero planes for bits = 1), per-row int64 sums of squared codes
    and nonzero counts, and an int32 flag word (QX_RF_NONFINITE on NaN).
    `bits` defaults to the narrowest field holding the quantiser's codes."""
    t = D.torch()
    if x.dtype not in (t.float32, t.float64):
        x = x.to(t.float64)
    bits = packed_bits(q) if bits is None else int(bits)
    if bits not in (1, 2, 4, 8):
        raise ValueError(f"no packed field holds codes of level bound {q.k}; use quantize_device")
    batch = x.shape[0] if x.dim() == 2 else 1
    n = x.shape[-1]
    L = N.load()
    words = L.qx_packed_words(n, bits)
    codes = t.empty((batch, words), dtype=t.int32, device=x.device)
    sums = t.zeros((2, batch), dtype=t.int64, device=x.device)
    flags = t.zeros(1, dtype=t.int32, device=x.device)
    nq, keep = native_quantizer(q)
    sig = D.signals(x)
    ctx = N.context(x.device.index)
    from ._call import call  # (status -> the reference's exception types)

    call(L.qx_quantize_packed, ctx, ctypes.byref(nq), ctypes.byref(sig), batch, bits, codes.data_ptr(),
         sums[0].data_ptr(), sums[1].data_ptr(), flags.data_ptr(), D.stream_handle())
    del keep
    return codes, sums[0], sums[1], flags


def unpack_codes(words: np.ndarray, n: int, bits: int) -> np.ndarray:
    """int64 codes of one packed row (the layout of qx_quantize_packed) on the
    host: a format decode for IntSignal, no quantisation."""
    b = np.ascontiguousarray(words).view(np.uint8)
    if bits == 8:
        return b.view(np.int8)[:n].astype(np.int64)
    if bits == 1:
        nw = (n + 31) // 32
        bb = np.unpackbits(b, bitorder="little")
        sgn, nz = bb[: 32 * nw][:n].astype(np.int64), bb[32 * nw:][:n].astype(np.int64)
        return nz * (1 - 2 * sgn)
    per = 8 // bits
    f = np.stack([(b >> (bits * k)) & ((1 << bits) - 1) for k in range(per)], axis=-1).reshape(-1)[:n]
    half = 1 << (bits - 1)
    return (f.astype(np.int64) ^ half) - half


def apply(q, s) -> IntSignal:
    """Quantise every stored sample; start and length preserved (quantize.py:105-107).

    The device writes bit-packed codes (2/4/8 bits for k <= 1/7/127), so the
    transfer back is n*b/8 bytes instead of 8n; the host only unpacks them."""
    samples = np.asarray(s.samples)
    if samples.dtype not in (np.float32, np.float64):
        samples = samples.astype(np.float64)
    bits = packed_bits(q)
    if not bits:
        codes = quantize_device(q, D.as_device(samples))
        return IntSignal(s.start, codes.cpu().numpy().reshape(-1), bound=q.k)
    words, _, _, _ = quantize_packed(q, D.as_device(samples), bits)
    return IntSignal(s.start, unpack_codes(words.cpu().numpy().reshape(-1), samples.shape[-1], bits), bound=q.k)
