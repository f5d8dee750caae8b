"""Probe: two independent half-size jobs (c4 shape, 5e7 queries each) scheduled sequentially on one
stream vs concurrently on two streams -- an upper bound on what overlapping the memory-bound sort
with the issue-bound DP could gain."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2409_14961_b200.scheduler import GpuScheduler
dev = torch.device("cuda:0")
jobs = []
for seed in (0, 1):
    inp, out, slo, cfg = W.c4(seed, n=50_000_000)
    g = GpuScheduler(len(inp), cfg, device=dev, per_batch=False)
    d = [torch.from_numpy(a.view(np.int32) if a.dtype != np.float32 else a).to(dev) for a in (inp, out, slo)]
    jobs.append((g, d))
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
for g, d in jobs:
    g.load(*d, s0)
torch.cuda.synchronize()

def seq():
    for g, d in jobs:
        g.schedule(s0); g.stats(s0)

def conc():
    jobs[0][0].schedule(s0); jobs[1][0].schedule(s1)
    jobs[0][0].stats(s0); jobs[1][0].stats(s1)

for name, fn in (("sequential", seq), ("concurrent", conc), ("sequential", seq), ("concurrent", conc)):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t) / 5 * 1e3, 3), "ms")
