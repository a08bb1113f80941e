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
           "native_quantizer", "thresholds"]


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


def apply(q, s) -> IntSignal:
    """Quantise every stored sample; start and length preserved (quantize.py:105-107)."""
    samples = np.asarray(s.samples, dtype=np.float64)
    codes = quantize_device(q, D.as_device(samples))
    return IntSignal(s.start, codes.cpu().numpy(), bound=q.k)
