"""Multi-rank host logic on the CPU: world_size-2 gloo process groups run the
same sharding + peak reduction the GPU ranks use, with the oracle standing in
for the per-rank kernels; the result must equal the unsharded oracle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_19974_b200 import parallel as PL


def test_shard_bounds_cover_exactly():
    for total in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [PL.shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_merge_peaks_semantics():
    assert PL.merge_peaks([(5, 10, 1), (7, 30, 2), (7, 20, 1)]) == (7, 20, 3)
    assert PL.merge_peaks([(3, 4, 0), (2, 9, 1)]) == (2, 9, 1)
    with pytest.raises(ValueError):
        PL.merge_peaks([(1, 1, 0)])


def test_merge_summaries_semantics():
    e = PL.SUMMARY_EMPTY
    assert PL.merge_summaries([(5, 10, 1, 0, 0, 0, 0, 0), (7, 30, 2, 1, 0, 0, 0, 0), (7, 20, 1, 0, 0, 1, 0, 0)]) == \
        (7, 20, 3, 1, 0, 0, 0, 0)
    assert PL.merge_summaries([e, (-4, -9, 2, 0, 1, 1, 0, 0)]) == (-4, -9, 2, 0, 1, 1, 0, 0)
    assert PL.merge_summaries([e, e]) == (0, 0, 0, 0, 0, 1, 0, 0)
    assert PL.merge_summaries([(3, 1, 1, 0, 0, 1, 1, 7), (3, 0, 1, 0, 0, 1, 1, 5)]) == (3, 0, 2, 0, 0, 1, 1, 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local(template, sl, qx, qy, lag_lo, lag_hi, s0):
    import oracle as O

    u = O.quantize(qx, template)
    v = O.quantize(qy, sl)
    first = s0 - (len(template) - 1)
    c = O.xcorr_bf(u, v, lag_lo - first, lag_hi - first)
    m, f, n = O.argmax(c)
    return m, lag_lo + f, n


def _worker(rank, world, port, seed, q, out):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(seed)
    stream = rng.laplace(size=3000).astype(np.float32)
    template = stream[1234:1234 + 200].copy()
    stream = stream + rng.normal(0, 0.3, stream.size).astype(np.float32)
    res = PL.template_search_sharded(template, stream, q, q, local_fn=_oracle_local)
    out.put((rank, res))
    dist.destroy_process_group()


def test_template_search_two_ranks_matches_unsharded():
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as O

    from paper_2509_19974_b200.quantize import sign

    q = sign()
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 11, q, out)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded oracle over the valid lags
    rng = np.random.default_rng(11)
    stream = rng.laplace(size=3000).astype(np.float32)
    template = stream[1234:1234 + 200].copy()
    stream = stream + rng.normal(0, 0.3, stream.size).astype(np.float32)
    u, v = O.quantize(q, template), O.quantize(q, stream)
    first = -(len(template) - 1)
    c = O.xcorr_bf(u, v, 0 - first, len(stream) - len(template) - first)
    m, f, n = O.argmax(c)
    assert got[0] == got[1] == (m, f, n)
    assert f == 1234


def _reduce_worker(rank, world, port, cases, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = []
    for case in cases:
        s = torch.tensor(case[rank], dtype=torch.int64)
        got.append(tuple(PL.reduce_summary(s).tolist()))
    out.put((rank, got))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_summary_reduction_protocol(world):
    """The two-round summary reduction (the device protocol of qx_dist.cu,
    here through gloo) equals merge_summaries on random per-rank summaries:
    negative and int64-extreme values, ties across ranks, empty shards and
    every flag."""
    rng = np.random.default_rng(world)
    cases = []
    for trial in range(40):
        ranks = []
        for r in range(world):
            if rng.random() < 0.2:
                ranks.append(PL.SUMMARY_EMPTY)
                continue
            v = int(rng.choice([-(1 << 62), -5, 0, 3, 7, (1 << 62)])) if trial % 2 else int(rng.integers(0, 3))
            lag = int(rng.integers(-(1 << 40), 1 << 40))
            ranks.append((v, lag, int(rng.integers(1, 4)), int(rng.random() < 0.1), int(rng.random() < 0.1),
                          int(rng.random() < 0.5), int(rng.random() < 0.1), int(rng.integers(0, 8))))
        cases.append(ranks)
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, port, cases, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, ranks in enumerate(cases):
        want = PL.merge_summaries(ranks)
        assert all(got[r][i] == want for r in range(world)), (i, ranks, [got[r][i] for r in range(world)], want)
