"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

The reference has no distributed code: its only parallelism is the thread
pool over accuracy trials (/root/reference/pkg/src/qxcorr/harness.py:301-305).
Here the units of work are sharded across GPUs and the samples never move
between them:

* Independent pairs (BASELINE configs 2 and 3): rank r takes the contiguous
  pair range ``shard_bounds(batch, r, world)``; there is no collective on the
  data path (``estimate_batch_sharded`` optionally all-gathers the 64-byte
  records afterwards: qx_estimate_batch_nccl).
* Long stream vs short template (config 5): the valid lags are split into
  ``world`` contiguous ranges; rank r correlates the template with its stream
  slice plus a (template - 1)-sample halo (``stream_shard``).  Each lag's sum
  uses only samples inside the slice, so the union of the per-rank summaries
  is the reference's argmax_set summary (estimator.py:50-57) of the
  unsharded correlogram.
* Config 4 (one long pair) is run as independent replicas (one pair per
  GPU): sharding the lag range of one full-lag NTT correlation needs every
  GPU to transform all of x and a window of y, so it cannot scale under a
  max-only collective; DESIGN.md says so.

The only collective is the summary reduction (``reduce_summary``), 8 int64
per rank in two rounds: MAX over {value, flags}, then one group of MAX
(smallest lag among the ranks holding the max) and SUM (their ties).  With
an NCCL group it runs inside the library on the device
(qx_summary_reduce_nccl / qx_template_search_nccl, torch's communicator);
with any other backend (gloo, the CPU tests) the same two rounds run through
torch.distributed.all_reduce (``_reduce_rounds``).
"""

from __future__ import annotations

import ctypes

import numpy as np

__all__ = ["shard_bounds", "stream_shard", "merge_peaks", "merge_summaries", "reduce_summary", "reduce_peak",
           "nccl_comm", "template_search_sharded", "estimate_batch_sharded", "SUMMARY_EMPTY"]

INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1
# summary layout (qx_template_search): value, lag, ties, nan, degx, degy_all, bad, badst
SUMMARY_EMPTY = (0, 0, 0, 0, 0, 1, 0, 0)


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of range(total) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def stream_shard(n_template: int, n_stream: int, rank: int, world: int):
    """Valid lags [lo, hi) of template-vs-stream owned by `rank`, and the
    stream slice [s0, s1) (with a template-1 halo) that covers them."""
    n_valid = n_stream - n_template + 1
    if n_valid < 1:
        raise ValueError("template longer than the stream")
    lo, hi = shard_bounds(n_valid, rank, world)
    return (lo, hi), (lo, hi - 1 + n_template)


def merge_peaks(peaks) -> tuple[int, int, int]:
    """Combine (value, lag, ties) summaries of disjoint lag ranges (host
    statement of the reduction's semantics).  Ranges with ties == 0 (empty)
    are ignored."""
    best = None
    for v, lag, t in peaks:
        if t == 0:
            continue
        if best is None or v > best[0]:
            best = [v, lag, t]
        elif v == best[0]:
            best[1] = min(best[1], lag)
            best[2] += t
    if best is None:
        raise ValueError("no lags in any shard")
    return tuple(best)


def merge_summaries(summaries) -> tuple:
    """The 8-word summaries of disjoint lag ranges -> the summary of their
    union (what reduce_summary computes across ranks)."""
    s = [tuple(int(v) for v in x) for x in summaries]
    live = [x for x in s if x[2]]
    v, lag, t = merge_peaks([x[:3] for x in live]) if live else (0, 0, 0)
    return (v, lag, t, max(x[3] for x in s), max(x[4] for x in s), min(x[5] for x in s), max(x[6] for x in s),
            max(x[7] for x in s))


def _reduce_rounds(summary, group=None):
    """The device protocol's two rounds through torch.distributed (any
    backend): `summary` is an int64[8] tensor on the backend's device,
    reduced in place."""
    import torch
    import torch.distributed as dist

    s = [int(v) for v in summary.cpu().tolist()]
    r1 = torch.tensor([s[0] if s[2] else INT64_MIN, s[3], s[4], s[6], s[7], 1 - s[5]], dtype=torch.int64,
                      device=summary.device)
    dist.all_reduce(r1, op=dist.ReduceOp.MAX, group=group)
    m = int(r1[0])
    holder = bool(s[2]) and s[0] == m
    lag_key = torch.tensor([-s[1] if holder else INT64_MIN], dtype=torch.int64, device=summary.device)
    ties = torch.tensor([s[2] if holder else 0], dtype=torch.int64, device=summary.device)
    dist.all_reduce(lag_key, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(ties, op=dist.ReduceOp.SUM, group=group)
    t = int(ties[0])
    r = r1.tolist()
    out = [m if t else 0, -int(lag_key[0]) if t else 0, t, r[1], r[2], 1 - r[5], r[3], r[4]]
    summary.copy_(torch.tensor(out, dtype=torch.int64))
    return summary


def _is_nccl(group) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "nccl"


def nccl_comm(group=None, device=None) -> int:
    """The ncclComm_t of a torch ProcessGroupNCCL (for the *_nccl C-ABI entry
    points); the communicator is created eagerly if needed."""
    import torch
    import torch.distributed as dist

    pg = group or dist.group.WORLD
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    backend = pg._get_backend(dev)
    ptr = backend._comm_ptr()
    if not ptr:  # lazily initialised communicator: one tiny collective creates it
        dist.barrier(group=pg, device_ids=[dev.index])
        ptr = backend._comm_ptr()
    return int(ptr)


def reduce_summary(summary, group=None):
    """In place: every rank's int64[8] summary (CUDA tensor for NCCL groups)
    -> the summary of the union of their lag ranges, on every rank."""
    from . import _device as D
    from . import _native as N
    from ._call import call

    if _is_nccl(group):
        ctx = N.context(summary.device.index)
        call(N.load().qx_summary_reduce_nccl, ctx, summary.data_ptr(), nccl_comm(group, summary.device),
             D.stream_handle())
        return summary
    host = summary.cpu()
    _reduce_rounds(host, group)
    summary.copy_(host)
    return summary


def reduce_peak(value: int, lag: int, ties: int, group=None, device=None) -> tuple[int, int, int]:
    """All ranks' (value, lag, ties) -> the global summary, on every rank."""
    import torch

    dev = device if device is not None and _is_nccl(group) else "cpu"
    s = torch.tensor([value, lag, ties, 0, 0, 0, 0, 0], dtype=torch.int64, device=dev)
    if not ties:
        s[5] = 1
    reduce_summary(s, group)
    v = s.tolist()
    if not v[2]:
        raise ValueError("no lags in any shard")
    return v[0], v[1], v[2]


def _raise_summary(s) -> tuple[int, int, int]:
    from ._call import raise_for
    from . import _native as N

    vmax, lmin, nties, nan, degx, degy, anybad, badst = (int(v) for v in s)
    if nan:
        raise ValueError("input contains NaN")
    if degx:
        raise_for(N.QX_DEGENERATE_QUANTIZATION, "x quantizes to all zeros")
    if degy:
        raise_for(N.QX_DEGENERATE_QUANTIZATION, "y quantizes to all zeros")
    if anybad:
        raise_for(int(badst), "template search block failed")
    return vmax, lmin, nties


def template_search_sharded(template, stream, qx, qy, group=None, device=None, local_fn=None, *,
                            stream_is_slice: bool = False, n_stream: int | None = None, stream_start: int = 0,
                            block: int | None = None, path: str = "auto") -> tuple[int, int, int]:
    """Peak summary of estimate(x=template, y=stream) over the valid lags,
    the stream split across the ranks of `group`; (value, lag, ties) on
    every rank, with the reference's exceptions.

    `stream` is the whole stream (each rank slices its share), or with
    `stream_is_slice` this rank's slice [s0, s1) of a stream of `n_stream`
    samples (stream_shard gives the bounds).  On an NCCL group the local
    search and the reduction are one C-ABI call (qx_template_search_nccl).
    `local_fn(template, slice, qx, qy, lag_lo, lag_hi, s0) -> (v, lag, ties)`
    replaces the GPU search (the CPU tests pass the oracle)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nt = len(template)
    ns = n_stream if stream_is_slice else len(stream)
    (lo, hi), (s0, s1) = stream_shard(nt, ns, rank, world)
    sl = stream if stream_is_slice else stream[s0:s1]
    if local_fn is not None:
        v, lag, t = local_fn(template, sl, qx, qy, lo, hi - 1, s0) if hi > lo else (0, 0, 0)
        s = torch.tensor([v, lag + stream_start, t, 0, 0, 0 if t else 1, 0, 0], dtype=torch.int64)
        if _is_nccl(group):
            s = s.to(device or torch.device("cuda", torch.cuda.current_device()))
        return _raise_summary(reduce_summary(s, group).tolist())
    from . import _device as D
    from . import _native as N
    from ._call import call
    from .batch import template_search_summary
    from .quantize import native_quantizer

    x = D.as_device(template).reshape(-1)
    y = D.as_device(sl).reshape(-1)
    if _is_nccl(group):
        out = torch.empty(8, dtype=torch.int64, device=x.device)
        nqx, _ = native_quantizer(qx)
        nqy, _ = native_quantizer(qy)
        sx, sy = D.signals(x, 0), D.signals(y, stream_start + s0)
        ctx = N.context(x.device.index)
        call(N.load().qx_template_search_nccl, ctx, ctypes.byref(sx), ctypes.byref(sy), ctypes.byref(nqx),
             ctypes.byref(nqy), 0 if block is None else int(block), N.PATHS[path], nccl_comm(group, x.device),
             out.data_ptr(), D.stream_handle())
        return _raise_summary(out.tolist())
    if hi > lo:
        s = template_search_summary(x, y, qx, qy, stream_start=stream_start + s0, block=block, path=path)
    else:
        s = torch.tensor(SUMMARY_EMPTY, dtype=torch.int64, device=x.device)
    return _raise_summary(reduce_summary(s, group).tolist())


def estimate_batch_sharded(x, y, qx, qy, group=None, *, lag_lo=None, lag_hi=None, gather: bool = True,
                           rows_are_local: bool = False, n_pairs: int | None = None, path: str = "auto"):
    """Independent pairs split across the ranks of `group` (configs 2/3):
    rank r estimates pairs shard_bounds(B, r, world) (`x`, `y` are the full
    batch, or with `rows_are_local` this rank's rows of an `n_pairs` batch).
    Returns (this rank's BatchResult, all records (B, 8) int64 or None).
    On NCCL with equal shards the gather is the library's ncclAllGather
    (qx_estimate_batch_nccl); otherwise torch's all_gather."""
    import torch
    import torch.distributed as dist

    from . import _device as D
    from . import _native as N
    from ._call import call
    from .batch import BatchResult, _bounds, estimate_batch
    from .quantize import native_quantizer

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    total = n_pairs if rows_are_local else x.shape[0]
    b0, b1 = shard_bounds(total, rank, world)
    xs = x if rows_are_local else x[b0:b1]
    ys = y if rows_are_local else y[b0:b1]
    xs, ys = D.as_device(xs), D.as_device(ys)
    equal = total % world == 0
    if gather and _is_nccl(group) and equal:
        nb = b1 - b0
        raw = torch.empty((nb, 8), dtype=torch.int64, device=xs.device)
        allr = torch.empty((total, 8), dtype=torch.int64, device=xs.device)
        nqx, _ = native_quantizer(qx)
        nqy, _ = native_quantizer(qy)
        sx, sy = D.signals(xs, 0), D.signals(ys, 0)
        lo, hi = _bounds(lag_lo, lag_hi)
        ctx = N.context(xs.device.index)
        call(N.load().qx_estimate_batch_nccl, ctx, ctypes.byref(sx), ctypes.byref(sy), nb, ctypes.byref(nqx),
             ctypes.byref(nqy), lo, hi, N.PATHS[path], raw.data_ptr(), nccl_comm(group, xs.device), allr.data_ptr(),
             D.stream_handle())
        return BatchResult(raw), allr
    mine = estimate_batch(xs, ys, qx, qy, lag_lo=lag_lo, lag_hi=lag_hi, path=path)
    if not gather:
        return mine, None
    per = -(-total // world)
    pad = torch.zeros((per, 8), dtype=torch.int64, device=mine.raw.device)
    pad[:b1 - b0] = mine.raw
    dev = pad.device if _is_nccl(group) else "cpu"
    pad = pad.to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    rows = [parts[r][:shard_bounds(total, r, world)[1] - shard_bounds(total, r, world)[0]] for r in range(world)]
    return mine, torch.cat(rows).to(mine.raw.device)
