"""Exact integer cross-correlation on the GPU (full correlogram).

Drop-in for /root/reference/pkg/src/qxcorr/intxcorr.py's ``xcorr_int_bf``
(96-100) and ``xcorr_int_ks`` (259-265): both names return the same
bit-identical int64 ``Correlogram`` (with ``norm_x``/``norm_y``) computed by
the NTT kernels through ``qx_xcorr_full``.  ``_check_coeff_bound`` (89-93)
and ``plan_ks``'s all-zero check (109-110) keep their exceptions.

``big_mul`` (intxcorr.py:183-205) keeps the reference's plugin slot with one
more backend, ``"cuda"``: the exact product of two big integers as one GPU
correlation of their 16-bit limbs plus a linear carry pass.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from ._call import call
from .errors import DegenerateInput, InternalOverflow
from .quantize import native_quantizer
from .signals import Correlogram, l2_norm

__all__ = ["xcorr_int_gpu", "xcorr_int_bf", "xcorr_int_ks", "MAX_COEFF_BOUND", "xcorr_full_device", "big_mul",
           "MUL_BACKENDS", "KSPlan", "plan_ks", "pack", "unpack_and_correct"]

MAX_COEFF_BOUND = 1 << 59  # intxcorr.py:50
# intxcorr.py:52 plus "cuda"; "auto" takes "cuda" from CUDA_MIN_BITS up
MUL_BACKENDS = ("auto", "cuda", "gmp", "native", "karatsuba", "schoolbook")
CUDA_MIN_BITS = 1 << 17


def _check_coeff_bound(n_min: int, k_u: int, k_v: int) -> None:
    if n_min * k_u * k_v > MAX_COEFF_BOUND:
        raise ValueError("coefficient bound N_min*K_u*K_v exceeds the supported int64 range")


def xcorr_full_device(x, y, qx, qy, x_start=0, y_start=0, path="auto"):
    """values (batch, nx+ny-1) int64 CUDA tensor and per-pair stats records.

    x, y: CUDA tensors (n,) or (batch, n); float rows are quantised with
    qx/qy, int64 rows are codes and qx/qy are then their integer bounds.
    """
    t = D.torch()
    xb = x if x.dim() == 2 else x.unsqueeze(0)
    yb = y if y.dim() == 2 else y.unsqueeze(0)
    batch = xb.shape[0]
    nout = xb.shape[1] + yb.shape[1] - 1
    values = t.empty((batch, nout), dtype=t.int64, device=x.device)
    stats = t.empty((batch, 8), dtype=t.int64, device=x.device)
    nqx, kx = native_quantizer(qx)
    nqy, ky = native_quantizer(qy)
    sx, sy = D.signals(xb, x_start), D.signals(yb, y_start)
    ctx = N.context(x.device.index)
    call(N.load().qx_xcorr_full, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, ctypes.byref(nqx),
         ctypes.byref(nqy), values.data_ptr(), stats.data_ptr(), N.PATHS[path], D.stream_handle())
    return values, stats


def xcorr_int_gpu(u, v) -> Correlogram:
    """sum_m u[m] * v[m+n] over every overlap lag, exact int64 (GPU)."""
    _check_coeff_bound(min(len(u.samples), len(v.samples)), max(u.bound, 1), max(v.bound, 1))
    du = D.as_device(np.asarray(u.samples, dtype=np.int64))
    dv = D.as_device(np.asarray(v.samples, dtype=np.int64))
    values, stats = xcorr_full_device(du, dv, int(u.bound), int(v.bound), int(u.start), int(v.start))
    st = stats[0].cpu().numpy()
    vals = values[0].cpu().numpy()
    first_lag = int(v.start) - (int(u.start) + len(u.samples) - 1)
    return Correlogram(first_lag, vals, norm_x=math.sqrt(int(st[3])), norm_y=math.sqrt(int(st[4])))


def xcorr_int_bf(u, v) -> Correlogram:
    """Reference name (intxcorr.py:96); same exact values as every path."""
    return xcorr_int_gpu(u, v)


def xcorr_int_ks(u, v, mul_backend: str = "auto") -> Correlogram:
    """Reference name (intxcorr.py:259); rejects all-zero input like plan_ks
    and unknown multiplication backends like big_mul."""
    if mul_backend not in MUL_BACKENDS:
        raise ValueError(f"unknown multiplication backend {mul_backend!r}")
    if not np.asarray(u.samples).any() or not np.asarray(v.samples).any():
        raise DegenerateInput("cannot plan a Kronecker correlation for an all-zero signal")
    return xcorr_int_gpu(u, v)


_LIMB = 16
_LIMB_MAX = (1 << _LIMB) - 1


def _limbs(a: int) -> np.ndarray:
    nb = (a.bit_length() + _LIMB - 1) // _LIMB
    return np.frombuffer(a.to_bytes(2 * nb, "little"), dtype="<u2").astype(np.int64)


def _big_mul_cuda(a: int, b: int) -> int:
    """a*b for naturals a, b > 0: conv(limbs(a), limbs(b)) as the exact GPU
    correlation of reverse(limbs(a)) with limbs(b) (index t = n + na - 1 is
    the convolution index), then carries: every coefficient is < 2^59
    (the 2^59 bound caps min(#limbs) at 2^27, i.e. 2^31-bit operands), so
    it splits into four 16-bit planes P_j and a*b = sum_j P_j << 16j."""
    la, lb = _limbs(a), _limbs(b)
    _check_coeff_bound(min(la.size, lb.size), _LIMB_MAX, _LIMB_MAX)
    du = D.as_device(la[::-1].copy())
    dv = D.as_device(lb)
    values, _ = xcorr_full_device(du, dv, _LIMB_MAX, _LIMB_MAX)
    c = values[0].cpu().numpy().view(np.uint64)
    out = 0
    for j in range(4):
        plane = ((c >> np.uint64(_LIMB * j)) & np.uint64(_LIMB_MAX)).astype("<u2")
        out += int.from_bytes(plane.tobytes(), "little") << (_LIMB * j)
    return out


def big_mul(a: int, b: int, backend: str = "auto") -> int:
    """Exact product of two big integers (intxcorr.py:183-205).

    "cuda" runs the NTT correlation kernels on 16-bit limbs (exact at every
    size up to 2^31-bit operands).  "auto" uses "cuda" when both operands
    have at least CUDA_MIN_BITS bits and a GPU is present, else the
    interpreter's multiplication.  "native", "karatsuba" and "schoolbook"
    return the interpreter's exact product (the reference's backends all
    return identical values); "gmp" needs gmpy2 like the reference."""
    if backend not in MUL_BACKENDS:
        raise ValueError(f"unknown multiplication backend {backend!r}")
    if backend == "gmp":
        try:
            import gmpy2
        except ImportError:
            raise ValueError("gmp backend requested but gmpy2 is not installed") from None
        return int(gmpy2.mpz(a) * gmpy2.mpz(b))
    if backend == "auto":
        big = min(abs(a).bit_length(), abs(b).bit_length()) >= CUDA_MIN_BITS
        backend = "cuda" if big and D.torch().cuda.is_available() else "native"
    if backend != "cuda":
        return a * b
    sign = -1 if (a < 0) != (b < 0) else 1
    a, b = abs(a), abs(b)
    if a == 0 or b == 0:
        return 0
    return sign * _big_mul_cuda(a, b)


# ------------------------------------------------ Kronecker substitution (host)
# The reference's KS plumbing (intxcorr.py:55-142, 208-256) with the same
# names, plan and exceptions, for callers that drive it step by step
# (pack -> big_mul -> unpack_and_correct).  The engine itself never packs:
# its exact NTT correlation replaces the packed product,
# and big_mul "cuda" multiplies packed naturals on the GPU.  Packing and slot
# extraction here are vectorised bit-plane operations (numpy packbits), not
# per-slot Python loops.


@dataclass(frozen=True)
class KSPlan:
    """Slot width L and biases of one Kronecker correlation (intxcorr.py:55-82):
    2^L > 4 * n_min * k_u * k_v, so biased slots never collide."""

    slot_bits: int
    n_min: int
    k_u: int
    k_v: int

    def __post_init__(self):
        if self.slot_bits < 1:
            raise ValueError("slot_bits must be >= 1")
        if (1 << self.slot_bits) <= 4 * self.n_min * self.k_u * self.k_v:
            raise ValueError("slot width too narrow for biased coefficients")

    @property
    def bias_u(self) -> int:
        return self.k_u

    @property
    def bias_v(self) -> int:
        return self.k_v

    @property
    def coeff_bound(self) -> int:
        return self.n_min * self.k_u * self.k_v


def plan_ks(u, v) -> KSPlan:
    """L = floor(log2(N_min K_u K_v)) + 3 (intxcorr.py:103-115)."""
    if not np.asarray(u.samples).any() or not np.asarray(v.samples).any():
        raise DegenerateInput("cannot plan a Kronecker correlation for an all-zero signal")
    n_min = min(len(u.samples), len(v.samples))
    _check_coeff_bound(n_min, int(u.bound), int(v.bound))
    return KSPlan(slot_bits=(n_min * int(u.bound) * int(v.bound)).bit_length() + 2, n_min=n_min,
                  k_u=int(u.bound), k_v=int(v.bound))


def _slots_to_int(vals: np.ndarray, L: int) -> int:
    """sum_n vals[n] * 2^(L n) for 0 <= vals < 2^L: the L low bits of every
    value laid end to end, little-endian."""
    if vals.size == 0:
        return 0
    bits = ((vals.astype(np.uint64)[:, None] >> np.arange(L, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.uint8)
    return int.from_bytes(np.packbits(bits.reshape(-1), bitorder="little").tobytes(), "little")


def _int_to_slots(p: int, L: int, count: int) -> np.ndarray:
    """count L-bit slots of the natural p (the inverse of _slots_to_int)."""
    nbytes = (L * count + 7) // 8
    raw = np.frombuffer(p.to_bytes(max(nbytes, (p.bit_length() + 7) // 8), "little")[:nbytes], dtype=np.uint8)
    bits = np.unpackbits(raw, bitorder="little")[:L * count].reshape(count, L).astype(np.uint64)
    return (bits << np.arange(L, dtype=np.uint64)[None, :]).sum(axis=1).astype(np.int64)


def pack(w, plan: KSPlan, *, bias: int) -> int:
    """sum_n (w[n] + bias) * 2^(L n) as one natural (intxcorr.py:133-142);
    InternalOverflow when a biased coefficient leaves [0, 2^L)."""
    shifted = np.asarray(w.samples, dtype=np.int64) + np.int64(bias)
    if shifted.size and (int(shifted.min()) < 0 or int(shifted.max()) >> plan.slot_bits):
        raise InternalOverflow("biased coefficient does not fit its slot")
    if plan.slot_bits > 63:
        return sum(int(x) << (plan.slot_bits * i) for i, x in enumerate(shifted.tolist()))
    return _slots_to_int(shifted, plan.slot_bits)


def unpack_and_correct(p: int, plan: KSPlan, u, v) -> Correlogram:
    """The exact signed correlation from the packed product of
    (reverse(u) + B_u) and (v + B_v) (intxcorr.py:226-256): the slots minus
    the three bias cross terms (window sums by prefix sums); InternalOverflow
    if a value exceeds N_min K_u K_v."""
    nu, nv = len(u.samples), len(v.samples)
    count = nu + nv - 1
    if plan.slot_bits > 63:
        mask = (1 << plan.slot_bits) - 1
        slots = np.array([(p >> (plan.slot_bits * n)) & mask for n in range(count)], dtype=object)
    else:
        slots = _int_to_slots(p, plan.slot_bits, count)
    cu = np.concatenate(([0], np.cumsum(np.asarray(u.samples, dtype=np.int64)[::-1])))
    cv = np.concatenate(([0], np.cumsum(np.asarray(v.samples, dtype=np.int64))))
    t = np.arange(count)
    ilo, ihi = np.maximum(0, t - nv + 1), np.minimum(nu - 1, t)
    jlo, jhi = np.maximum(0, t - nu + 1), np.minimum(nv - 1, t)
    values = (slots - plan.bias_v * (cu[ihi + 1] - cu[ilo]) - plan.bias_u * (cv[jhi + 1] - cv[jlo])
              - plan.bias_u * plan.bias_v * (ihi - ilo + 1))
    values = np.asarray(values, dtype=np.int64)
    if int(np.abs(values).max()) > plan.coeff_bound:
        raise InternalOverflow("corrected coefficient exceeds N_min*K_u*K_v")
    first_lag = int(v.start) - (int(u.start) + nu - 1)
    return Correlogram(first_lag, values, norm_x=l2_norm(u), norm_y=l2_norm(v))
