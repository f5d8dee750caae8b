UELLM_PIPE_TRACE=1 python - <<'PY' 2>&1 | tail -60
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import workloads as W
from paper_2409_14961_b200 import uellm as U
inp, out, slo, cfg = W.c4(0)
n = len(inp); c = U.make_config(cfg)
p_in = torch.from_numpy(inp.view(np.int32)).pin_memory(); p_out = torch.from_numpy(out.view(np.int32)).pin_memory(); p_slo = torch.from_numpy(slo).pin_memory()
h_order = torch.empty(n, dtype=torch.int32).pin_memory(); h_offs = torch.empty(n + 1, dtype=torch.int32).pin_memory()
nb = np.zeros(1, np.uint64); tot = U.Totals(); st = torch.cuda.Stream()
for groups in (12,):
    wsb = U.pipeline_workspace_bytes(n, c, groups); ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    for it in range(2):
        t = time.perf_counter()
        U.schedule_pipelined(n, p_in, p_out, p_slo, c, groups, ws, wsb, h_order, h_offs, nb, ctypes.addressof(tot), st)
        print("groups", groups, "call_ms", (time.perf_counter() - t) * 1e3, flush=True)
    del ws; torch.cuda.empty_cache()
PY
