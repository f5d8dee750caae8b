#!/usr/bin/env python
"""PCIe floor of the end-to-end (host-buffer) step: plain pinned copies of exactly the bytes the
e2e step moves -- the three 4 B/query input arrays host->device and order (4 B/query) + batch
offsets (4 B/batch) device->host -- timed with CUDA events, no GPU work in between.
usage: python tools/pcie_floor.py [n] [batches]   (c4: 1e8 queries, 2.64e6 batches)"""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 2_642_654
dev = torch.device("cuda:0")
h_in = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(3)]
d_in = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3)]
d_out = [torch.empty(n, dtype=torch.int32, device=dev), torch.empty(m + 1, dtype=torch.int32, device=dev)]
h_out = [torch.empty(n, dtype=torch.int32).pin_memory(), torch.empty(m + 1, dtype=torch.int32).pin_memory()]
st, st2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("h2d_inputs", lambda: [d.copy_(h, non_blocking=True) for d, h in zip(d_in, h_in)]),
                 ("d2h_outputs", lambda: [h.copy_(d, non_blocking=True) for h, d in zip(h_out, d_out)])):
    with torch.cuda.stream(st):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 5
# both directions at once (H2D and D2H on two streams, the pipelined call overlaps them)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
st2.wait_event(e0)
for _ in range(5):
    with torch.cuda.stream(st):
        [d.copy_(h, non_blocking=True) for d, h in zip(d_in, h_in)]
    with torch.cuda.stream(st2):
        [h.copy_(d, non_blocking=True) for h, d in zip(h_out, d_out)]
st.wait_stream(st2)
e1.record(st)
torch.cuda.synchronize()
res["both_overlapped"] = e0.elapsed_time(e1) / 5
h2d_b, d2h_b = 12 * n, 4 * n + 4 * (m + 1)
print(json.dumps({"n": n, "batches": m, "h2d_bytes": h2d_b, "d2h_bytes": d2h_b,
                  "ms": res, "h2d_gbs": h2d_b / res["h2d_inputs"] / 1e6, "d2h_gbs": d2h_b / res["d2h_outputs"] / 1e6,
                  "floor_ms": max(res["h2d_inputs"], res["both_overlapped"]),
                  "note": "pinned host memory, CUDA events on the copy stream, mean of 5 after 2 warm-ups"}))
