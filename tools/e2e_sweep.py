"""e2e experiment: uellm_schedule_pipelined on c4 for several group counts, the PCIe copy floor
(pinned H2D of the 12 B/query inputs, D2H of order + offsets) and the fixed per-call overhead."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2409_14961_b200 import uellm as U

dev = torch.device("cuda:0")
inp, out, slo, cfg = W.c4(0)
n = len(inp)
c = U.make_config(cfg)
p_in = torch.from_numpy(inp.view(np.int32)).pin_memory()
p_out = torch.from_numpy(out.view(np.int32)).pin_memory()
p_slo = torch.from_numpy(slo).pin_memory()
h_order = torch.empty(n, dtype=torch.int32).pin_memory()
h_offs = torch.empty(n + 1, dtype=torch.int32).pin_memory()
nb = np.zeros(1, np.uint64)
tot = U.Totals()
st = torch.cuda.Stream()


def timed(fn, k=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3


d_in = torch.empty(n, dtype=torch.int32, device=dev)
d_out = torch.empty(n, dtype=torch.int32, device=dev)
d_slo = torch.empty(n, dtype=torch.float32, device=dev)
d_ord = torch.empty(n, dtype=torch.int32, device=dev)


def h2d():
    with torch.cuda.stream(st):
        d_in.copy_(p_in, non_blocking=True); d_out.copy_(p_out, non_blocking=True); d_slo.copy_(p_slo, non_blocking=True)
    st.synchronize()


def d2h():
    with torch.cuda.stream(st):
        h_order.copy_(d_ord, non_blocking=True)
        h_offs[:2_700_000].copy_(d_ord[:2_700_000], non_blocking=True)
    st.synchronize()


print("h2d_ms", round(timed(h2d), 3), "d2h_ms", round(timed(d2h), 3))
for groups in (10, 12, 16, 20, 24):
    wsb = U.pipeline_workspace_bytes(n, c, groups)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    ms = timed(lambda: U.schedule_pipelined(n, p_in, p_out, p_slo, c, groups, ws, wsb, h_order, h_offs, nb,
                                            ctypes.addressof(tot), st))
    print("groups", groups, "e2e_ms", round(ms, 3), "m", int(nb[0]))
    del ws
    torch.cuda.empty_cache()
# fixed per-call overhead: one small window
small = 10_000
c2 = U.make_config(cfg.replace(window=small))
wsb = U.pipeline_workspace_bytes(small, c2, 1)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
ms = timed(lambda: U.schedule_pipelined(small, p_in[:small], p_out[:small], p_slo[:small], c2, 1, ws, wsb, h_order,
                                        h_offs, nb, ctypes.addressof(tot), st), k=20)
print("small_call_ms", round(ms, 3))
