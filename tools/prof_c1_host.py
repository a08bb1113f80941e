import cProfile, pstats, sys, os, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W
x, y = W.c1(0)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
q = P.sign()
for _ in range(50): P.estimate_batch(xd, yd, q, q)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500): P.estimate_batch(xd, yd, q, q)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"issue {1e6*(t1-t0)/500:.1f} us/call, with drain {1e6*(t2-t0)/500:.1f} us/call")
pr = cProfile.Profile(); pr.enable()
for _ in range(500): P.estimate_batch(xd, yd, q, q)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
