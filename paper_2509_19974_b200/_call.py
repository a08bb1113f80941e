"""Native calls with the reference's exception semantics (status -> exception,
include/qxcorr_b200.h qx_status)."""

from __future__ import annotations

from . import _native as N
from .errors import DegenerateInput, DegenerateQuantization, InternalOverflow

_MAP = {
    N.QX_ERR_INVALID: ValueError,
    N.QX_DEGENERATE_QUANTIZATION: DegenerateQuantization,
    N.QX_DEGENERATE_INPUT: DegenerateInput,
    N.QX_BOUND_EXCEEDED: ValueError,
    N.QX_INTERNAL_OVERFLOW: InternalOverflow,
    N.QX_ERR_UNSUPPORTED: NotImplementedError,
    N.QX_ERR_NONFINITE: ValueError,
}


def raise_for(status: int, message: str):
    exc = _MAP.get(status, RuntimeError)
    raise exc(message)


def call(fn, ctx, *args) -> None:
    st = fn(ctx, *args)
    if st != N.QX_OK:
        msg = N.load().qx_context_last_error(ctx).decode() or N.load().qx_status_string(st).decode()
        raise_for(st, msg)
