"""Small end-to-end run of every entry point, for compute-sanitizer (T6 in SURVEY.md section 4):
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py
c1 / c2 shapes, forced small DP tiles (fix-up + cascade), uniform stretches (deferred fills,
traceback exit maps), reload, Alg. 1, FIFO, simulator, profiler stand-ins (both paths), HELR and the
pipelined host-buffer call.  Prints SANITIZE_RUN_OK at the end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2409_14961_b200 import uellm as U
from paper_2409_14961_b200.scheduler import GpuScheduler

dev = torch.device("cuda:0")


def run(inp, out, slo, cfg):
    g = GpuScheduler(len(inp), cfg, device=dev)
    g.run(torch.from_numpy(inp.view(np.int32)).to(dev), torch.from_numpy(out.view(np.int32)).to(dev),
          torch.from_numpy(slo).to(dev))
    g.simulate(torch.from_numpy(W.poisson_arrivals(len(inp), 1, 3000).view(np.int64)).to(dev))
    torch.cuda.synchronize()
    return g


run(*W.c1(0, lam=10**6))
inp, out, slo, cfg = W.c2(1, n=3000)
run(inp, out, slo, cfg.replace(dp_tile=128))
run(inp, out, slo, cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.05, threshold=400.0))
run(inp, out, slo, cfg.replace(mode=W.MODE_FIFO))
inp, out, slo, cfg = W.c3(2, n=20_000)
run(inp, out, W.gen_uniform_slo(20_000, 2), cfg.replace(window=7000))
t = torch.from_numpy(W.true_output_lengths(20_000, 3).view(np.int32)).to(dev)
p = torch.zeros(20_000, dtype=torch.int32, device=dev)
for levels in (True, False):
    st = U.MonitorState()
    st.inflation_factor = 1.0
    s = torch.frombuffer(bytearray(bytes(st)), dtype=torch.uint8).to(dev)
    pc = U.make_predictor(W.PredictorConfig(window=3000))
    wsb = U.predict_workspace_bytes(20_000, pc) if levels else 0
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device=dev)
    U.predict_lengths(20_000, t, pc, s, p, None, None, ws if wsb else None, wsb)
# uniform stretches over many tiles: deferred periodic fills (k_dp_fill), traceback exit maps and
# parallel re-marking (k_trace_maps / k_trace_remark)
inp, out, slo, cfg = W.uniform_runs(5, n=60_000, runs=((14_000, 128, 257), (9_000, 64, 513)))
run(inp, out, slo, cfg.replace(dp_tile=1024))
# asynchronous reload into the same profile (device-side validation, status word)
inp, out, slo, cfg = W.c2(3, n=4000)
g = run(inp, out, slo, cfg.replace(window=1000))
perm = np.random.default_rng(1).permutation(4000)
g.reload(torch.from_numpy(inp[perm].view(np.int32)).to(dev), torch.from_numpy(out[perm].view(np.int32)).to(dev),
         torch.from_numpy(slo[perm]).to(dev))
g.schedule()
g.stats()
torch.cuda.synchronize()
assert int(g.status_word().item()) == 0
topo = W.random_topology(3, 6)
wsb = U.helr_workspace_bytes(6)
U.helr_plan(topo, torch.zeros(wsb, dtype=torch.uint8, device=dev), wsb)
# host-buffer pipelined call (two compute lanes, copy streams)
inp, out, slo, cfg = W.c3(4, n=30_000)
cfg = cfg.replace(window=5000)
c = U.make_config(cfg)
wsb = U.pipeline_workspace_bytes(30_000, c, 3)
ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
tot = U.Totals()
U.schedule_pipelined(30_000, inp, out, slo, c, 3, ws, wsb, np.zeros(30_000, np.uint32), np.zeros(30_001, np.uint32),
                     np.zeros(1, np.uint64), ctypes.addressof(tot))
torch.cuda.synchronize()
print("SANITIZE_RUN_OK")
