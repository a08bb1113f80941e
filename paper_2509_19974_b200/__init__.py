"""B200-native quantise -> exact integer cross-correlation -> argmax engine.

A drop-in for the hot path of the reference package ``qxcorr``
(arxiv 2509.19974; /root/reference/pkg/src/qxcorr): the same function names,
argument meanings and exceptions, with the arithmetic in hand-written sm_100a
kernels behind the C ABI include/qxcorr_b200.h (libqxcorr_b200.so).

    from paper_2509_19974_b200 import Signal, sign, estimate
    r = estimate(Signal(0, x), Signal(0, y), sign(), sign())

Batched, windowed and streaming entry points (new): ``estimate_batch``,
``estimate_batch_host``, ``template_search``; multi-GPU sharding in
``parallel``.
"""

from . import accuracy, ingest, parallel
from .batch import (BatchResult, EstimatePlan, check_results, estimate_batch, estimate_batch_host, estimate_sweep,
                    estimate_sweep_host, template_search)
from .errors import (
    BadLength,
    ConfigError,
    DegenerateInput,
    DegenerateQuantization,
    InternalOverflow,
    ParseError,
    QxcorrError,
    UnsupportedFormat,
)
from .estimator import EstimationResult, argmax_set, estimate, estimate_real
from .intxcorr import (MUL_BACKENDS, KSPlan, big_mul, pack, plan_ks, unpack_and_correct, xcorr_int_bf, xcorr_int_gpu,
                       xcorr_int_ks)
from .quantize import (Quantizer, apply, custom, from_spec, packed_bits, quantize_packed, random_monotone, sign,
                       uniform, unpack_codes)
from .realxcorr import xcorr_real_at, xcorr_real_bf, xcorr_real_fft
from .signals import Correlogram, IntSignal, Signal, add, crop, l2_norm, reverse, scale, shift, trim

__version__ = "0.1.0"

__all__ = [
    "QxcorrError", "DegenerateInput", "DegenerateQuantization", "InternalOverflow", "BadLength",
    "ParseError", "UnsupportedFormat", "ConfigError",
    "Signal", "IntSignal", "Correlogram", "reverse", "shift", "l2_norm", "trim", "scale", "add", "crop",
    "Quantizer", "sign", "uniform", "custom", "from_spec", "apply", "random_monotone", "quantize_packed",
    "unpack_codes", "packed_bits",
    "KSPlan", "plan_ks", "pack", "unpack_and_correct",
    "xcorr_int_gpu", "xcorr_int_bf", "xcorr_int_ks", "xcorr_real_at", "xcorr_real_bf", "xcorr_real_fft", "big_mul",
    "MUL_BACKENDS",
    "EstimationResult", "argmax_set", "estimate", "estimate_real",
    "BatchResult", "EstimatePlan", "estimate_batch", "estimate_batch_host", "estimate_sweep", "estimate_sweep_host", "check_results", "template_search",
    "accuracy", "ingest", "parallel",
]
