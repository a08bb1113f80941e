"""How the pinned host buffers behind the C2 e2e are allocated changes the
PCIe rate: time the sweep's copies alone (QX_SWEEP_COMPUTE=0) and the full
e2e call from (1) torch pin_memory(), (2) an empty pinned tensor filled
afterwards, (3) anonymous 2-MiB-aligned memory advised MADV_HUGEPAGE and
registered with cudaHostRegister.  Usage: python tools/pinned_probe.py"""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19974_b200 as P  # noqa: E402
from paper_2509_19974_b200 import _native, workloads as W  # noqa: E402

xs, ys, lag = W.c2()
qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in (1, 2, 4, 8)]
sweep = [(q, q) for q in qs]
est = 4 * xs.shape[0]
libc = ctypes.CDLL("libc.so.6", use_errno=True)
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None


def huge_pinned(a):
    size = (a.nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    buf = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    al = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(size), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer((ctypes.c_char * size).from_address(al), dtype=a.dtype, count=a.size).reshape(a.shape)
    arr[...] = a
    rc = torch.cuda.cudart().cudaHostRegister(al, size, 0)
    return arr, buf, rc


def time_calls(hx, hy, env, reps=12):
    _native.set_option("sweep_compute", int(env.get("QX_SWEEP_COMPUTE", 1)))
    for _ in range(2):
        P.estimate_sweep_host(hx, hy, sweep)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = P.estimate_sweep_host(hx, hy, sweep)
        ts.append(time.perf_counter() - t0)
    _native.set_option("sweep_compute", 1)
    if not env:
        for r in res:
            assert np.array_equal(r["lag"], lag)
    return 1e3 * float(np.median(ts))


def report(name, hx, hy):
    c = time_calls(hx, hy, {"QX_SWEEP_COMPUTE": "0"})
    e = time_calls(hx, hy, {})
    print(f"{name:34s} copy-only {c:.3f} ms ({(xs.nbytes + ys.nbytes) / c / 1e6:.1f} GB/s)   e2e {e:.3f} ms"
          f" -> {est / e * 1e3:.0f} est/s", flush=True)


if os.environ.get("BENCHLIKE"):
    import torch.distributed  # noqa: F401

    torch.cuda.set_device(0)
    xd0 = torch.from_numpy(xs).to("cuda")
    if os.environ.get("BENCHLIKE") == "2":
        torch.cuda.synchronize()
torch.cuda.init()
t1x, t1y = torch.from_numpy(xs).pin_memory(), torch.from_numpy(ys).pin_memory()
report("torch pin_memory()", t1x.numpy(), t1y.numpy())
t2x = torch.empty(xs.shape, dtype=torch.float32, pin_memory=True)
t2y = torch.empty(ys.shape, dtype=torch.float32, pin_memory=True)
t2x.numpy()[...] = xs
t2y.numpy()[...] = ys
report("torch.empty(pin_memory=True)", t2x.numpy(), t2y.numpy())
hx, bx, rx = huge_pinned(xs)
hy, by, ry = huge_pinned(ys)
print("cudaHostRegister rc", rx, ry)
report("MADV_HUGEPAGE + cudaHostRegister", hx, hy)
thp = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
print("THP:", thp)
report("torch pin_memory() again", t1x.numpy(), t1y.numpy())

if os.environ.get("STAGES"):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench as B

    hxn, hyn = t1x.numpy(), t1y.numpy()
    with B.ClockSampler(0):
        time.sleep(0.5)
    report("after ClockSampler", hxn, hyn)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    report("after device allocations", hxn, hyn)
    for _ in range(40):
        flush.zero_()
        P.estimate_sweep(xd, yd, sweep)
    torch.cuda.synchronize()
    report("after 40 device sweeps", hxn, hyn)
    from paper_2509_19974_b200 import _native

    with _native.profile(timed=True):
        for _ in range(10):
            for q in qs:
                P.estimate_batch(xd, yd, q, q)
        torch.cuda.synchronize()
    report("after a timed profile", hxn, hyn)
    report("device=0", hxn, hyn)
