"""Benchmark: BASELINE.json's metric on its configuration 2 (bit-depth sweep).

One step = the hot path (quantise -> exact full-lag integer cross-correlation
-> argmax) over the whole C2 batch at every bit depth: 64 float32 pairs of
2^18 samples at b = 1, 2, 4, 8, i.e. 256 lag estimates.  Inputs are seeded
synthetic data with BASELINE's shapes and statistics (workloads.c2); they are
resident in HBM before timing (`value`) or copied from pinned host memory
inside the timed region through the C ABI's host entry point (`e2e`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]

Under torchrun every rank processes its own 64-pair batch (weak scaling; the
pairs are independent, so there is no data-path collective); the timed region
is bracketed by a barrier + synchronize and the max over ranks is reported.
`--impl reference` times the reference algorithm's CPU implementation (the C
oracle: float64 quantise, Kronecker substitution with GMP, argmax; all host
threads) on a bounded sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lag estimates/sec (quantize+int xcorr+argmax)"
UNIT = "estimates/s"
BITS = (1, 2, 4, 8)
L2_BYTES = 126 * (1 << 20)
E2E_WARM = 60  # e2e warm-up calls (see the e2e block in main)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE config (default c2, the headline; the others: tools/bench_run.py)")
    ap.add_argument("--pairs", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs (other_configs)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_desc(pairs, world):
    from paper_2509_19974_b200 import workloads as W

    return {"workload": "BASELINE config 2: bit-depth sweep", "pairs_per_gpu": pairs, "n": W.C2_N,
            "bits": list(BITS), "lags": "full -(N-1)..(N-1)", "dtype_in": "float32",
            "quantizers": "b=1 sign(); b>=2 uniform(2^(b-1)-1, 6*sigma/2^b)",
            "estimates_per_step": pairs * len(BITS) * world,
            "l2": "flushed between timed steps (512 MiB write), per-step CUDA events",
            "parallelism": f"pairs x{world} ranks (weak)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            self.nv = None
            self.err = str(exc)

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- CPU (oracle)
def cpu_arm(pairs_sample, threads, xs, ys, min_seconds=0.0):
    """Reference algorithm on the host: the C oracle (quantise in float64,
    Kronecker substitution + GMP multiply, argmax) for every bit depth on
    `pairs_sample` pairs, threaded over pairs, repeated until `min_seconds`
    of work.  Returns (estimates/s, seconds, passes)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    from paper_2509_19974_b200 import workloads as W

    O.build()
    qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in BITS]
    t0 = time.perf_counter()
    n_est = passes = 0
    while True:
        for q in qs:
            rec = O.estimate_batch_f32(xs[:pairs_sample], ys[:pairs_sample], q, q, threads=threads)
            n_est += len(rec)
        passes += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    return n_est / dt, dt, passes


def _cpu_info():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_baselines

    return cpu_baselines.cpu_info()


def reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2509_19974_b200 import workloads as W

    threads = os.cpu_count() or 1
    sample = args.pairs  # the same 64-pair, 4-depth workload as the GPU arm's step
    xs, ys, lag = W.c2(pairs=sample)
    times = []
    for i in range(args.warmup + args.steps):
        rate, dt, _ = cpu_arm(sample, threads, xs, ys)
        if i >= args.warmup:
            times.append(dt)
    per_step = sum(times) / len(times)
    value = sample * len(BITS) / per_step
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded, BASELINE config 2 shapes)",
            "config": config_desc(sample, 1) | {"sample": f"{sample} pairs x 4 bit depths per step"},
            "same_config": True,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} pairs x {len(BITS)} bit depths of config 2 per step"} | _cpu_info(),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    if args.config != "c2":
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_run

        return bench_run.run_reference(args) if args.impl == "reference" else bench_run.run(args)
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    import paper_2509_19974_b200 as P
    from paper_2509_19974_b200 import _native, workloads as W

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    pairs = args.pairs
    xs, ys, lag = W.c2(pairs=pairs, first=rank * pairs)
    xd = torch.from_numpy(xs).to(dev)
    yd = torch.from_numpy(ys).to(dev)
    qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in BITS]
    out_all = torch.empty((len(BITS), pairs, 8), dtype=torch.int64, device=dev)
    outs = list(out_all)
    sweep_q = [(q, q) for q in qs]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        # one C-ABI call: the 4 bit depths on concurrent compute lanes
        P.estimate_sweep(xd, yd, sweep_q, out=out_all)

    def step_serial():
        # the same work one bit depth after another on the current stream
        # (the per-kernel profile: launch durations without overlap)
        for q, o in zip(qs, outs):
            P.estimate_batch(xd, yd, q, q, out=o)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness of the benchmarked work: every estimate equals the pinned
    # oracle's exact (peak, smallest lag, ties) and code norms
    # (tests/golden/fullsize.*: pairs 0..511, i.e. every rank's batch up to 8 GPUs)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fullsize_golden as G

    for bi, o in enumerate(outs):
        G.check_c2(bi, rank * pairs, o.cpu().numpy().view(_native.RESULT_DTYPE).reshape(-1))

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # timed region: launches are counted (no per-launch events, no gaps)
    with ClockSampler(local) as clk, _native.profile(timed=False) as prof:
        for a, b in evs:
            flush.zero_()
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # separate run with every library launch bracketed by CUDA events on its
    # stream: per-kernel device time for the roofline of the dominant kernel
    kprof_steps = min(args.steps, 10)
    with _native.profile(timed=True) as kprof:
        for _ in range(kprof_steps):
            flush.zero_()
            step_serial()
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    est_per_step = pairs * len(BITS) * world
    value = est_per_step * args.steps / (total_ms / 1e3)
    samples_per_step = est_per_step * 2 * W.C2_N
    ms_per_step = total_ms / args.steps

    # dominant kernel and its roofline, from the event-timed run (kprof_steps)
    P2 = 1 << 19
    n_pairs_total = pairs * len(BITS) * kprof_steps
    alg_bytes = {  # compulsory bytes of each kernel over the profiled steps (prime 0)
        "ntt_pass1": n_pairs_total * (2 * W.C2_N * 4 + 2 * P2 * 4),  # floats in, Y out
        "ntt_pass2": n_pairs_total * (3 * P2 * 4),                  # Y_u, Y_v in, Z out
        "ntt_pass3": n_pairs_total * (P2 * 4),                      # Z in
    }
    bflies = {"ntt_pass1": n_pairs_total * 2 * (P2 // 2) * 10, "ntt_pass2": n_pairs_total * 3 * (P2 // 2) * 9,
              "ntt_pass3": n_pairs_total * (P2 // 2) * 10}
    kinds = kprof.result
    total_ms_prof = sum(m for _, m in kinds.values())
    dom = max(kinds, key=lambda k: kinds[k][1])
    dom_ms = kinds[dom][1]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes.get(dom, 0) / (dom_ms / 1e3) / 1e9 if dom_ms else None
    traffic = None
    ncu_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu_path):
        traffic = json.load(open(ncu_path)).get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s",
            "kernel_ms_share": dom_ms / total_ms_prof if total_ms_prof else None,
            "timing": f"CUDA events around each launch on its stream, {kprof_steps} steps after the timed region, "
                      "the bit depths one after another (no lane overlap)"}
    int_peak_path = os.path.join(ROOT, "profiles", "int_peaks.json")
    int_roof = {"kernel": dom, "butterflies_per_s": bflies.get(dom, 0) / (dom_ms / 1e3) if dom_ms else None}
    if os.path.exists(int_peak_path):
        ip = json.load(open(int_peak_path))
        if ip.get("butterflies_per_s"):
            int_roof["peak"] = ip["butterflies_per_s"]
            int_roof["frac"] = int_roof["butterflies_per_s"] / ip["butterflies_per_s"]
    all_bfly = sum(bflies.values())
    ntt_ms = sum(kinds[k][1] for k in bflies if k in kinds)
    int_roof["all_ntt_butterflies_per_s"] = all_bfly / (ntt_ms / 1e3) if ntt_ms else None
    if "peak" in int_roof and int_roof["all_ntt_butterflies_per_s"]:
        int_roof["all_ntt_frac"] = int_roof["all_ntt_butterflies_per_s"] / int_roof["peak"]
    # SURVEY 8(d) accounting: 3 (P/2) log2 P butterflies per pair and bit depth
    # (956,301,312 per 64-pair depth at P = 2^19) over the measured step time,
    # against the butterfly peak and against the FMA-pipe bounds of a Shoup
    # butterfly (1 IMAD.HI + 2 IMAD; pure IMAD rate / 3 as the looser one)
    s8d = pairs * len(BITS) * 3 * (P2 // 2) * int(math.log2(P2))  # one rank's step
    int_roof["s8d_butterflies_per_step"] = s8d
    int_roof["s8d_butterflies_per_s"] = s8d / (ms_per_step / 1e3)
    if os.path.exists(int_peak_path):
        ip = json.load(open(int_peak_path))
        if ip.get("butterflies_per_s"):
            int_roof["s8d_frac"] = int_roof["s8d_butterflies_per_s"] / ip["butterflies_per_s"]
        if ip.get("imad_per_s") and ip.get("imad_hi_per_s"):
            fma_bound = 1.0 / (1.0 / ip["imad_hi_per_s"] + 2.0 / ip["imad_per_s"])
            int_roof["fma_pipe_bound_butterflies_per_s"] = fma_bound
            int_roof["s8d_frac_of_fma_pipe_bound"] = int_roof["s8d_butterflies_per_s"] / fma_bound
            int_roof["imad_rate_bound_butterflies_per_s"] = ip["imad_per_s"] / 3.0
            int_roof["s8d_frac_of_imad_rate_bound"] = int_roof["s8d_butterflies_per_s"] / (ip["imad_per_s"] / 3.0)

    # e2e through the C ABI host entry point (pinned host buffers, H2D+D2H inside)
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(xs).pin_memory()
        hy = torch.from_numpy(ys).pin_memory()
        hxn, hyn = hx.numpy(), hy.numpy()
        n_e2e = max(10, args.steps // 3)
        sweep = [(q, q) for q in qs]
        # warm-up: lane streams, arenas and staging reach their steady size,
        # and freshly pinned host buffers reach their steady DMA rate -- the
        # first ~40 copies from a new pinned allocation run up to 30% slower
        # (tools/e2e_series.py, profiles/r01_e2e_series.txt)
        for _ in range(E2E_WARM):
            P.estimate_sweep_host(hxn, hyn, sweep, device=local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        call_s = []
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            tc = time.perf_counter()
            res = P.estimate_sweep_host(hxn, hyn, sweep, device=local)
            call_s.append(time.perf_counter() - tc)
        t1 = time.perf_counter()
        e2e_s = torch.tensor([t1 - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        for bi, r in enumerate(res):
            G.check_c2(bi, rank * pairs, r)
        # the bound e2e is held to: the same call with its kernels skipped
        # (option sweep_compute=0: the chunked pinned H2D copies, joins and the
        # results D2H alone), wall-clock per call like e2e
        with _native.option("sweep_compute", 0, device=local):
            P.estimate_sweep_host(hxn, hyn, sweep, device=local)
            tb = time.perf_counter()
            for _ in range(n_e2e):
                P.estimate_sweep_host(hxn, hyn, sweep, device=local)
            h2d_s = (time.perf_counter() - tb) / n_e2e
        # and with its copies skipped (option sweep_restage=0: the staging buffer
        # already holds these inputs): the same schedule's compute alone
        with _native.option("sweep_restage", 0, device=local):
            tb = time.perf_counter()
            for _ in range(n_e2e):
                P.estimate_sweep_host(hxn, hyn, sweep, device=local)
            comp_s = (time.perf_counter() - tb) / n_e2e
        # the same call from PAGEABLE numpy arrays (what a reference caller using
        # INTEGRATION.md section 3 passes): the driver stages them synchronously
        xs_pg, ys_pg = np.array(xs, copy=True), np.array(ys, copy=True)
        P.estimate_sweep_host(xs_pg, ys_pg, sweep, device=local)
        tb = time.perf_counter()
        for _ in range(n_e2e):
            rp = P.estimate_sweep_host(xs_pg, ys_pg, sweep, device=local)
        pageable_s = (time.perf_counter() - tb) / n_e2e
        for bi, r in enumerate(rp):
            G.check_c2(bi, rank * pairs, r)
        e2e_val = est_per_step * n_e2e / float(e2e_s.item())
        e2e = {"value": e2e_val, "unit": UNIT,
               "call_ms": {"median": 1e3 * statistics.median(call_s), "min": 1e3 * min(call_s),
                           "max": 1e3 * max(call_s)},
               "h2d_gbs": (xs.nbytes + ys.nbytes) / h2d_s / 1e9,
               "copy_only_ms": 1e3 * h2d_s, "compute_only_ms": 1e3 * comp_s,
               "h2d_bound": {"value": est_per_step / h2d_s, "frac": e2e_val / (est_per_step / h2d_s),
                             "what": "estimates/s if each step cost only its copies (the same call, kernels skipped)"},
               "pageable": {"value": est_per_step / pageable_s, "call_ms": 1e3 * pageable_s,
                            "what": "the same call from pageable numpy arrays (no pinning by the caller)"},
               "h2d_bytes_per_step": int(xs.nbytes + ys.nbytes),
               "d2h_bytes_per_step": int(len(BITS) * pairs * 64), "steps": n_e2e, "warmup_calls": E2E_WARM,
               "path": "qx_estimate_sweep_host (C ABI, pinned host buffers; inputs staged once per step "
                       "in 8-pair chunks on a copy stream, the 4 bit depths of each chunk on 4 concurrent "
                       "compute lanes)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = min(pairs, max(8, threads))
        rate, dt, passes = cpu_arm(sample, threads, xs, ys, min_seconds=10.0)
        import cpu_baselines as CB

        fft = CB.fft_pairs(xs, ys, threads, min_seconds=8.0, max_pairs=threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{passes} passes over {sample} pairs x {len(BITS)} bit depths of config 2 ({dt:.1f} s): "
                         "C oracle = reference algorithm (float64 quantise, KS + GMP mpn_mul, argmax)",
               "fft": {"value": fft["value"], "unit": UNIT, "cores": threads, "kind": "port",
                       "sample": fft["sample"] + f" ({fft['seconds']:.1f} s): the reference's Real-FFT path "
                                 "(realxcorr.py:99-116 restated in oracle/refport.py), one estimate per pair "
                                 "(independent of the bit depth)"}} | CB.cpu_info()

    # the other BASELINE configs on this GPU (rank 0 of a single-GPU run):
    # each checked against its planted delay, failures reported, not fatal
    other = None
    if rank == 0 and world == 1 and not args.no_configs:
        other = {}
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs
        for name in ("c1", "c1batch", "c3full", "c4", "c5"):
            try:
                other.update(bench_configs.run([name]))
            except Exception as exc:  # keep the headline line
                other[name] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32 mod-p NTT (exact int64 results)",
                "data": "synthetic (seeded numpy, BASELINE config 2 shapes/SNR); inputs resident in HBM",
                "config": config_desc(pairs, world),
                "gsamples_per_s": samples_per_step * args.steps / (total_ms / 1e3) / 1e9,
                "gpu_launches": prof.launches,
                "step": "qx_estimate_sweep: one C-ABI call per step, the 4 bit depths on 4 concurrent compute "
                        "lanes (streams with their own scratch) joined to the timing stream",
                "kernels": {k: {"launches": c, "ms_per_step": m / kprof_steps} for k, (c, m) in kinds.items()},
                "roofline": roof, "int_roofline": int_roof, "clocks": clk.summary(), "e2e": e2e,
                "cpu_baseline": cpu, "step_ms_median": statistics.median(step_ms),
                "other_configs": other}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
