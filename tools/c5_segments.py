#!/usr/bin/env python
"""Per-segment stage times of BJ configs[4] (c5): each of the four 2.5 M-query segments run as its
own job (10^6-query windows), stage events + diagnostics.  usage: python tools/c5_segments.py [K]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2409_14961_b200 import uellm as U  # noqa: E402
from paper_2409_14961_b200.scheduler import GpuScheduler  # noqa: E402


def run(name, inp, out, slo, cfg, K, dev, stream):
    d_in = torch.from_numpy(inp.view(np.int32)).to(dev)
    d_out = torch.from_numpy(out.view(np.int32)).to(dev)
    d_slo = torch.from_numpy(slo).to(dev)
    g = GpuScheduler(len(inp), cfg, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in U.STAGES]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for e in ev:
        e.record(stream)
    acc = {}
    for k in range(K + 1):
        t0.record(stream)
        g.load(d_in, d_out, d_slo, stream)
        U.set_stage_events(g.profile, ev)
        g.schedule(stream)
        g.stats(stream)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        if k == 0:
            continue
        st = {"total": t0.elapsed_time(t1)}
        for a, b, nm in [(0, 1, "sort"), (1, 2, "decode"), (2, 3, "dp_local"), (3, 4, "dp_fix"),
                         (4, 5, "dp_cascade"), (5, 6, "traceback"), (6, 7, "compact"), (8, 9, "stats")]:
            st[nm] = ev[a].elapsed_time(ev[b])
        for kk, v in st.items():
            acc[kk] = acc.get(kk, 0.0) + v / K
    diag = g.diagnostics(stream)
    print(json.dumps({"segment": name, "n": len(inp), "ms": {k: round(v, 4) for k, v in acc.items()},
                      "diag": diag}), flush=True)


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    inp, out, slo, cfg = W.c5(0)
    n = len(inp)
    q = n // 4
    names = ["i_identical", "ii_all_violating", "iii_over_cap", "iv_anti_sorted"]
    run("c5_all", inp, out, slo, cfg, K, dev, stream)
    for s in range(4):
        a, b = s * q, (s + 1) * q if s < 3 else n
        run(names[s], inp[a:b], out[a:b], slo[a:b], cfg, K, dev, stream)


if __name__ == "__main__":
    main()
