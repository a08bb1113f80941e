"""Multi-rank sharding with the real kernels (GPU): two processes on one GPU,
joined by a gloo group, each searching ITS shard of the full-size config-5
stream (2^28 samples, its valid-lag range plus the (template-1)-sample halo,
uploaded alone) on the tensor cores; the summary reduction then combines the
two ranks.  Both ranks must return the single-GPU answer, which is the pinned
oracle's (tests/golden/fullsize.json).  The ranks' kernels never wait on each
other (the reduction runs on the host through gloo), so sharing one GPU is
safe; on several GPUs the same code takes the NCCL path."""

import json
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _c5_rank(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2509_19974_b200 as P
    from paper_2509_19974_b200 import parallel as PL
    from paper_2509_19974_b200 import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tpl, st, off, sn2 = W.c5()
    (lo, hi), (s0, s1) = PL.stream_shard(len(tpl), len(st), rank, world)
    td = torch.from_numpy(tpl).cuda()
    sd = torch.from_numpy(st[s0:s1]).cuda()  # only this rank's slice (+ halo) on the device
    res = {}
    for b in (1, 2):
        if b == 1:
            qa = qb = P.sign()
        else:
            qa, qb = P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + sn2))
        res[b] = PL.template_search_sharded(td, sd, qa, qb, stream_is_slice=True, n_stream=len(st))
        res[f"local{b}"] = P.template_search(td, sd, qa, qb, stream_start=s0)
    out.put((rank, (lo, hi), res))
    dist.destroy_process_group()


def test_two_ranks_c5_full_size_on_one_gpu():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize.json")))["c5"]
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_rank, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = [out.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort()
    assert got[0][1][0] == 0 and got[0][1][1] == got[1][1][0] and got[1][1][1] == g["stream"] - g["template"] + 1
    for case in g["cases"]:
        want = (case["peak"], case["lag"], case["ties"])
        b = case["b"]
        assert got[0][2][b] == got[1][2][b] == want, (b, got)
        # the shard holding the planted lag has the peak; the other a smaller max
        holder = 0 if want[1] < got[0][1][1] else 1
        assert got[holder][2][f"local{b}"] == want and got[1 - holder][2][f"local{b}"][0] < want[0]
