"""bench.py --config c1|c3|c4|c5: BASELINE.json's metric on its other
configurations, under the same contract as the C2 headline (one process per
GPU under torchrun, W warm-up steps, K timed steps bracketed by a barrier +
synchronize, CUDA events, the max over ranks, clocks sampled in the timed
region, every result checked against the pinned oracle's full-size records,
e2e through the public host API, roofline of the dominant kernel, the
reference's CPU paths beside it).

Scaling per config:
* c3: 65,536 pairs split across the ranks (strong scaling, no collective);
* c5: the 2^28-sample stream split across the ranks by valid-lag range with a
  (template - 1)-sample halo, one summary reduction (strong scaling; NCCL
  inside the library for N > 1);
* c1, c4: one pair per rank, independent replicas (weak scaling): a single
  pair does not shard (C1: microseconds; C4: lag-sharding one NTT needs every
  GPU to transform all of x).
"""

from __future__ import annotations

import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

METRIC = "lag estimates/sec and Gsamples/s (quantize+int xcorr+argmax)"
FP4_MACS_PER_CLK_SM = 16336.0  # profiles/r01_tc_fp4.txt (tools/tc_fp4.cu, M128 x N>=128 kind::mxf4)
I8_MACS_PER_CLK_SM = 8190.0    # profiles/r01_tc_rate.json (tools/tc_rate.cu)
CLK = 1.965e9


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    pk = json.load(open(p)) if os.path.exists(p) else {}
    return pk.get("hbm_gbs", 6550.4), ("MEASURED_PEAKS.json hbm_gbs" if pk else "fallback 6550.4 GB/s")


def _int_peak():
    return json.load(open(os.path.join(ROOT, "profiles", "int_peaks.json")))


class Workload:
    name = ""
    unit = "estimates/s"
    scaling = "weak"
    flush = False  # inputs smaller than L2: flush between steps

    def desc(self) -> dict:
        raise NotImplementedError


# ------------------------------------------------------------------ C1
class C1(Workload):
    name = "c1"
    flush = True

    def setup(self, P, W, torch, rank, world, dev):
        self.P, self.W = P, W
        self.x, self.y = W.c1(0)
        self.xd, self.yd = torch.from_numpy(self.x).to(dev), torch.from_numpy(self.y).to(dev)
        self.out = torch.empty((1, 8), dtype=torch.int64, device=dev)
        self.units = world  # one estimate per rank and step
        self.dev = dev
        # the low-latency serving form of estimate_batch (qx_plan_run: one C-ABI call per estimate)
        self.plan = P.EstimatePlan(self.xd, self.yd, P.sign(), P.sign())

    def step(self):
        self.plan(self.xd, self.yd, out=self.out)

    def check(self, G):
        r = self.out.cpu().numpy().view(_result_dtype()).reshape(-1)[0]
        G.check_c1(int(r["lag"]), int(r["value"]))

    def e2e_step(self):
        # the serving form from host rows: one qx_plan_run_host call per pair (both rows read from
        # page-locked buffers over PCIe by the popc launch itself, the 64-B result written to a mapped
        # page-locked buffer, one synchronisation)
        if not hasattr(self, "xh"):
            import torch
            self.xh = torch.from_numpy(self.x).pin_memory().numpy()
            self.yh = torch.from_numpy(self.y).pin_memory().numpy()
            self.rh = np.zeros(1, dtype=_result_dtype())
        return self.plan.run_host(self.xh, self.yh, out=self.rh)

    def e2e_pageable(self):
        return self.P.estimate_batch_host(self.x, self.y, self.P.sign(), self.P.sign(), device=self.dev.index)

    def e2e_bytes(self):
        return self.x.nbytes + self.y.nbytes, 64

    def roofline(self, kinds, hbm):
        ms = sum(m for _, m in kinds.values())
        n = sum(c for c, _ in kinds.values())
        pk = _int_peak()["popc_per_s"]
        words = (1 << 14) * (2 * (1 << 14) - 1) / 32  # popc words of the full-lag window
        ach = words / (ms / n / 1e3) if ms else None
        return {"bound": "popc", "kernel": "popc", "achieved": ach, "peak": pk, "unit": "popc-words/s",
                "frac": ach / pk if ach else None, "traffic": None,
                "note": "single pair: latency-bound (one cooperative launch); achieved = 2^14 x (2^15-1) / 32 "
                        "popc-words per launch / the event-timed launch duration"}

    def cpu(self, CB, cores):
        ti = CB.int_single(self.x.astype(np.float64), self.y.astype(np.float64), self.P.sign(), self.P.sign())
        tf = CB.fft_single(self.x.astype(np.float32), self.y.astype(np.float32))
        return {"value": 1.0 / ti, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": "one C1 estimate on 1 core: float64 quantise, KS + GMP mpn_mul, argmax",
                "fft": {"value": 1.0 / tf, "unit": self.unit, "cores": 1, "kind": "port",
                        "sample": "one ccf_fft_array (float32, radix-2 numpy, realxcorr.py:99-116) + argmax"}}

    def desc(self):
        return {"workload": "BASELINE config 1: single 2^14 float64 pair, sign(), full lags", "n": 1 << 14,
                "lags": "full", "parallelism": "replicas (one pair per GPU)", "l2": "flushed between timed steps"}


def _result_dtype():
    from paper_2509_19974_b200 import _native as N

    return N.RESULT_DTYPE


# ------------------------------------------------------------------ C3
class C3(Workload):
    name = "c3"
    scaling = "strong"

    def setup(self, P, W, torch, rank, world, dev):
        from paper_2509_19974_b200 import parallel as PL

        self.P, self.W, self.torch = P, W, torch
        self.b0, self.b1 = PL.shard_bounds(W.C3_PAIRS, rank, world)
        a0 = self.b0 // 1024 * 1024
        xs, ys, _ = W.c3(pairs=self.b1 - a0, first=a0)
        xs, ys = xs[self.b0 - a0:], ys[self.b0 - a0:]
        self.hx = torch.from_numpy(np.ascontiguousarray(xs)).pin_memory()
        self.hy = torch.from_numpy(np.ascontiguousarray(ys)).pin_memory()
        self.xd, self.yd = self.hx.to(dev), self.hy.to(dev)
        self.qs = [W.bit_quantizer(b, W.C3_SIGMA) for b in (2, 4)]
        nb = self.b1 - self.b0
        self.outs = [torch.empty((nb, 8), dtype=torch.int64, device=dev) for _ in self.qs]
        self.units = 2 * W.C3_PAIRS  # both bit depths of every pair, whole job
        self.dev = dev

    def step(self):
        for q, o in zip(self.qs, self.outs):
            self.P.estimate_batch(self.xd, self.yd, q, q, lag_lo=-512, lag_hi=512, out=o)

    def check(self, G):
        for bi, o in enumerate(self.outs):
            G.check_c3(bi, self.b0, o.cpu().numpy().view(_result_dtype()).reshape(-1))

    def e2e_step(self):
        return self.P.estimate_sweep_host(self.hx.numpy(), self.hy.numpy(), [(q, q) for q in self.qs], lag_lo=-512,
                                          lag_hi=512, device=self.dev.index)

    def e2e_bytes(self):
        return self.hx.numel() * 4 + self.hy.numel() * 4, 2 * (self.b1 - self.b0) * 64

    def roofline(self, kinds, hbm):
        c, ms = kinds.get("direct", (0, 0.0))
        nb = self.b1 - self.b0
        alg = nb * 2 * self.W.C3_N * 4  # floats read once per launch
        ach = alg / (ms / c / 1e3) / 1e9 if c else None
        return {"bound": "hbm", "kernel": "direct (tcgen05 kind::i8 window)", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm if ach else None, "traffic": _ncu_traffic("direct"),
                "algorithmic_bytes_per_launch": alg}

    def cpu(self, CB, cores):
        xs, ys = self.hx.numpy()[:256], self.hy.numpy()[:256]
        n = self.W.C3_N
        t_lo, t_hi = n - 1 - 512, n - 1 + 512
        ints = [CB.int_pairs(xs, ys, q, q, cores, min_seconds=4.0, t_lo=t_lo, t_hi=t_hi, max_pairs=8 * cores)
                for q in self.qs]
        fft = CB.fft_pairs(xs, ys, cores, min_seconds=4.0, max_pairs=8 * cores)
        rate = 2.0 / sum(1.0 / r["value"] for r in ints)
        return {"value": rate, "unit": self.unit, "cores": cores, "kind": "port",
                "sample": f"b=2 and b=4 estimates on {ints[0]['sample']} (full KS correlogram sliced to -512..512)",
                "fft": {"value": fft["value"], "unit": self.unit, "cores": cores, "kind": "port",
                        "sample": fft["sample"]}}

    def desc(self):
        return {"workload": "BASELINE config 3: 65,536 pairs x 4096 float32, lags -512..512, b = 2, 4",
                "pairs": self.W.C3_PAIRS, "n": self.W.C3_N, "bits": [2, 4],
                "parallelism": "pairs sharded over ranks (strong scaling, no collective)",
                "l2": "inputs (2 GiB) larger than L2"}


# ------------------------------------------------------------------ C4
class C4(Workload):
    name = "c4"
    unit = "Gsamples/s"

    def setup(self, P, W, torch, rank, world, dev):
        self.P, self.W = P, W
        x, y, _ = W.c4()
        self.hx, self.hy = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
        self.xd, self.yd = self.hx.to(dev), self.hy.to(dev)
        self.q = W.bit_quantizer(4, W.C4_SIGMA)
        self.out = torch.empty((1, 8), dtype=torch.int64, device=dev)
        self.units = world * 2 * W.C4_N / 1e9  # Gsamples per step, whole job
        self.dev = dev

    def step(self):
        self.P.estimate_batch(self.xd, self.yd, self.q, self.q, out=self.out)

    def check(self, G):
        G.check_c4(self.out.cpu().numpy().view(_result_dtype()).reshape(-1)[0])

    def e2e_step(self):
        return self.P.estimate_batch_host(self.hx.numpy(), self.hy.numpy(), self.q, self.q, device=self.dev.index)

    def e2e_bytes(self):
        return self.hx.numel() * 8, 64

    def roofline(self, kinds, hbm):
        P = 1 << 25
        bfl = 3 * (P // 2) * 25
        ms = sum(m for k, (c, m) in kinds.items() if k.startswith("ntt") or k == "other")
        steps = max(1, kinds.get("ntt_pass2", (1, 0))[0])
        pk = _int_peak()["butterflies_per_s"]
        ach = bfl / (ms / steps / 1e3) if ms else None
        return {"bound": "int (NTT butterflies)", "kernel": "all NTT passes (outer + four-step)", "achieved": ach,
                "peak": pk, "unit": "butterflies/s", "frac": ach / pk if ach else None, "traffic": None,
                "note": "3 (P/2) log2 P butterflies, P = 2^25, per estimate / the event-timed NTT time; peak = "
                        "profiles/int_peaks.json (measured DIF butterfly loop)"}

    def cpu(self, CB, cores):
        x, y = self.hx.numpy(), self.hy.numpy()
        ti = CB.int_single(x, y, self.q, self.q)
        n_s = 1 << 22
        tf = CB.fft_single(x[:n_s].copy(), y[:n_s].copy(), scale_to=self.W.C4_N)
        gs = 2 * self.W.C4_N / 1e9
        return {"value": gs / ti, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"one full C4 estimate (2^24 pair, b=4) on 1 core in {ti:.1f} s: float64 quantise, KS + GMP "
                          "mpn_mul, argmax",
                "fft": {"value": gs / tf, "unit": self.unit, "cores": 1, "kind": "port",
                        "sample": "ccf_fft_array + argmax timed on the first 2^22 samples of x and y, extrapolated by "
                                  "P log2 P to P = 2^25"}}

    def desc(self):
        return {"workload": "BASELINE config 4: one 2^24 float32 Laplacian pair, 0 dB, b = 4, full lags (NTT P=2^25)",
                "n": self.W.C4_N, "parallelism": "replicas (one pair per GPU)",
                "l2": "inputs (128 MiB) and NTT scratch larger than L2"}


# ------------------------------------------------------------------ C5
class C5(Workload):
    name = "c5"
    unit = "Gsamples/s"
    scaling = "strong"

    def setup(self, P, W, torch, rank, world, dev):
        from paper_2509_19974_b200 import parallel as PL

        self.P, self.W, self.torch, self.PL = P, W, torch, PL
        tpl, st, off, sn2 = W.c5()
        self.ns = st.size
        (self.lo, self.hi), (s0, s1) = PL.stream_shard(tpl.size, st.size, rank, world)
        self.s0 = s0
        self.ht = torch.from_numpy(tpl).pin_memory()
        self.hs = torch.from_numpy(np.ascontiguousarray(st[s0:s1])).pin_memory()
        del st
        self.td, self.sd = self.ht.to(dev), self.hs.to(dev)
        self.qs = [(P.sign(), P.sign()),
                   (P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + sn2)))]
        self.world = world
        self.units = 2 * self.ns / 1e9  # stream samples searched per step (both bit depths), whole job
        self.res = [None, None]
        self.dev = dev

    def _search(self, t, s, qa, qb):
        if self.world == 1:
            return self.P.template_search(t, s, qa, qb)
        return self.PL.template_search_sharded(t, s, qa, qb, stream_is_slice=True, n_stream=self.ns)

    def step(self):
        for i, (qa, qb) in enumerate(self.qs):
            if self.world == 1:
                self.res[i] = self.P.batch.template_search_summary(self.td, self.sd, qa, qb)
            else:
                self.res[i] = self._search(self.td, self.sd, qa, qb)

    def check(self, G):
        for i, b in enumerate((1, 2)):
            r = self.res[i]
            r = tuple(int(v) for v in r.tolist()[:3]) if hasattr(r, "tolist") else r
            G.check_c5(b, r)

    def e2e_step(self):
        return [self._search(self.ht, self.hs, qa, qb) for qa, qb in self.qs]

    def e2e_bytes(self):
        return 2 * (self.hs.numel() + self.ht.numel()) * 4, 2 * 64

    def roofline(self, kinds, hbm):
        # one search = one main-block launch + one remainder-block launch over the rank's valid
        # lags; the work of a search is divided by the summed time of all its launches
        c, ms = kinds.get("direct_f4", (0, 0.0))
        searches = self.ksteps * len(self.qs)
        macs = 4096 * (self.hi - self.lo)
        peak = FP4_MACS_PER_CLK_SM * 148 * CLK * 2 / 1e12
        ach = 2 * macs / (ms / searches / 1e3) / 1e12 if c else None
        return {"bound": "tensor", "kernel": "direct_f4 (tcgen05 kind::mxf4 template search)", "achieved": ach,
                "peak": peak, "unit": "TFLOP/s", "frac": ach / peak if ach else None, "traffic": _ncu_traffic("direct_f4"),
                "launches_per_search": c / searches if c else None,
                "note": "2 x 4096 x (valid lags of the rank) flops per search / the event-timed launches of one search; peak = the "
                        "measured kind::mxf4 rate 16,336 MACs/clk/SM x 148 SMs x 1.965 GHz (profiles/r01_tc_fp4.txt)"}

    def cpu(self, CB, cores):
        t = self.ht.numpy()
        st = self.hs.numpy()
        ints = [CB.int_stream(t, st, qa, qb, cores, nblocks=4 * cores) for qa, qb in self.qs]
        fft = CB.fft_stream(t, st, cores, min_seconds=4.0, nblocks=2 * cores)
        rate = 2.0 / sum(1.0 / r["samples_per_s"] for r in ints) / 1e9
        return {"value": rate, "unit": self.unit, "cores": cores, "kind": "port",
                "sample": f"b=1 and b=2 on {ints[0]['sample']}",
                "fft": {"value": fft["samples_per_s"] / 1e9, "unit": self.unit, "cores": cores, "kind": "port",
                        "sample": fft["sample"]}}

    def desc(self):
        return {"workload": "BASELINE config 5: 4096-sample template vs 2^28-sample float32 stream, valid lags, b = 1, 2",
                "stream": self.ns, "template": 4096,
                "parallelism": "stream sharded by valid-lag range with (template-1)-sample halos; one summary reduction",
                "l2": "stream (1 GiB) larger than L2"}


def _ncu_traffic(kind):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get("kernels", {}).get(kind, {}).get("dram_bytes_per_launch")


WORKLOADS = {"c1": C1, "c3": C3, "c4": C4, "c5": C5}


def run(args):
    import torch
    import torch.distributed as dist

    import paper_2509_19974_b200 as P
    import paper_2509_19974_b200.batch  # noqa: F401
    from paper_2509_19974_b200 import _native, workloads as W

    import bench as B
    import cpu_baselines as CB
    import fullsize_golden as G

    rank, world, local = B.dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = WORKLOADS[args.config]()
    wl.setup(P, W, torch, rank, world, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if wl.flush else None
    for _ in range(max(args.warmup, 3)):
        wl.step()
    torch.cuda.synchronize()
    wl.check(G)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with B.ClockSampler(local) as clk, _native.profile(timed=False) as prof:
        for a, b in evs:
            if flush is not None:
                flush.zero_()
            a.record()
            wl.step()
            b.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wl.check(G)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = wl.units * args.steps / (total_ms / 1e3)
    # per-kernel device time (every library launch bracketed by events on its stream)
    ksteps = min(args.steps, 5)
    with _native.profile(timed=True) as kprof:
        for _ in range(ksteps):
            if flush is not None:
                flush.zero_()
            wl.step()
        torch.cuda.synchronize()
    hbm, hbm_src = _peaks()
    wl.ksteps = ksteps
    roof = wl.roofline(kprof.result, hbm)
    roof["peak_source"] = hbm_src if roof.get("unit") == "GB/s" else roof.get("note", "")
    # e2e: the public host API with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # C1 is one 50-us call per step: warm up past the first calls on fresh page-locked
        # buffers (slower, as in the C2 line's e2e) and time enough calls for a stable mean
        for _ in range(60 if wl.name == "c1" else 3):
            wl.e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 10)) if wl.name != "c1" else max(200, args.steps)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            wl.e2e_step()
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        hb, db = wl.e2e_bytes()
        e2e = {"value": wl.units * n_e2e / float(dt.item()), "unit": wl.unit, "h2d_bytes_per_step": int(hb),
               "d2h_bytes_per_step": int(db), "steps": n_e2e, "path": "public host API, pinned host buffers"}
        if wl.name == "c1":
            e2e["path"] = ("EstimatePlan.run_host (qx_plan_run_host): page-locked rows read in place over PCIe "
                           "(zero-copy), the record written to a mapped page-locked buffer, one synchronisation")
            e2e["h2d_bytes_per_step"] = int(hb)  # read by the kernel over PCIe, no staging copy
        if hasattr(wl, "e2e_pageable"):
            # the same estimate from pageable numpy rows (a caller that does not pin)
            for _ in range(3):
                wl.e2e_pageable()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                wl.e2e_pageable()
            torch.cuda.synchronize()
            e2e["pageable"] = {"value": wl.units * n_e2e / (time.perf_counter() - t0),
                               "what": "estimate_batch_host from pageable numpy rows"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        cpu = wl.cpu(CB, cores) | CB.cpu_info()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": wl.scaling, "vs_baseline": None, "dtype": "int (exact integer correlation)",
                "data": "synthetic (seeded numpy, BASELINE shapes/SNR); inputs resident in HBM",
                "config": wl.desc() | {"world": world}, "gpu_launches": prof.launches,
                "kernels": {k: {"launches": c, "ms_per_step": m / ksteps} for k, (c, m) in kprof.result.items()},
                "roofline": roof, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
                "step_ms_median": statistics.median(step_ms),
                "checked": "every result equals the pinned oracle's full-size record (tests/golden/fullsize.*)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    """--impl reference --config cX: the reference's CPU path (the oracle
    port of Integer-KS, all host threads) on a bounded sample of the config,
    rank 0 only."""
    import bench as B
    import cpu_baselines as CB

    rank, world, local = B.dist_env()
    if rank != 0:
        return
    from paper_2509_19974_b200 import workloads as W

    import paper_2509_19974_b200 as P

    cores = os.cpu_count() or 1
    times, unit, sample = [], "estimates/s", ""
    for i in range(args.warmup + args.steps):
        if args.config == "c1":
            x, y = W.c1(0)
            dt, units, unit = CB.int_single(x, y, P.sign(), P.sign()), 1.0, "estimates/s"
            sample = "one C1 estimate (1 core)"
        elif args.config == "c3":
            if i == 0:
                xs, ys, _ = W.c3(pairs=1024)
            q2, q4 = W.bit_quantizer(2, W.C3_SIGMA), W.bit_quantizer(4, W.C3_SIGMA)
            n = 4 * cores
            t0 = time.perf_counter()
            for q in (q2, q4):
                CB.int_pairs(xs, ys, q, q, cores, min_seconds=0.0, t_lo=W.C3_N - 513, t_hi=W.C3_N + 511,
                             max_pairs=n)
            dt, units = time.perf_counter() - t0, 2.0 * n
            sample = f"{n} pairs x 2 bit depths per step ({cores} threads)"
        elif args.config == "c4":
            if i == 0:
                x, y, _ = W.c4()
            dt, units, unit = CB.int_single(x, y, W.bit_quantizer(4, W.C4_SIGMA), W.bit_quantizer(4, W.C4_SIGMA)), \
                2 * W.C4_N / 1e9, "Gsamples/s"
            sample = "one full C4 estimate (1 core)"
        else:
            if i == 0:
                tpl, st, off, sn2 = W.c5()
            r = [CB.int_stream(tpl, st, P.sign(), P.sign(), cores, nblocks=2 * cores),
                 CB.int_stream(tpl, st, P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + sn2)),
                               cores, nblocks=2 * cores)]
            dt = sum(x["seconds"] for x in r)
            units, unit = 2 * (2 * cores) * (1 << 18) / 1e9, "Gsamples/s"
            sample = f"2 x {2 * cores} blocks of 2^18 valid lags per step ({cores} threads)"
        if i >= args.warmup:
            times.append(dt / units)
    value = 1.0 / statistics.mean(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded, BASELINE shapes)", "config": {"workload": args.config, "sample": sample},
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample}
            | CB.cpu_info(),
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
