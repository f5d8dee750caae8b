"""Torch-facing convenience layer over the C ABI: owns a device workspace and output buffers
for up to n queries and runs load -> schedule -> stats on one CUDA stream.  PyTorch is used
only for device memory and streams."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import uellm as U


class GpuScheduler:
    def __init__(self, n: int, cfg, device=None, per_batch: bool = True):
        self.device = torch.device(device or "cuda")
        self.cfg = U.make_config(cfg)
        self.n = int(n)
        self.ws_bytes = U.workspace_bytes(self.n, self.cfg)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        if self.ws.data_ptr() % 256:
            raise RuntimeError("workspace not 256-byte aligned")
        m = max(self.n, 1)
        self.order = torch.empty(m, dtype=torch.int32, device=self.device)      # u32 bits
        self.offsets = torch.empty(self.n + 1, dtype=torch.int32, device=self.device)
        self.num_batches = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.per_batch = (torch.empty((m, 80), dtype=torch.uint8, device=self.device)
                          if per_batch else None)
        self.totals = torch.empty(U.TOTALS_BYTES, dtype=torch.uint8, device=self.device)
        self.profile = None

    # -- the three ABI steps, device-resident -------------------------------------------
    def load(self, input_len, pred_out_len, slo_s, stream=None):
        n = int(input_len.shape[0])
        if n != self.n:
            raise ValueError(f"scheduler sized for {self.n} queries, got {n}")
        self.profile = U.profile_load(n, input_len, pred_out_len, slo_s, self.cfg, self.ws,
                                      self.ws_bytes, stream)
        return self.profile

    def reload(self, input_len, pred_out_len, slo_s, stream=None):
        """Asynchronous load of the next n queries (device tensors) into the current profile; the
        validation verdict lands in the device status word (status())."""
        if self.profile is None:
            raise RuntimeError("reload needs a profile from load()")
        U.profile_reload(self.profile, input_len, pred_out_len, slo_s, self.cfg, stream)
        return self.profile

    def status_word(self):
        """The profile's device status word as a 1-element int32 tensor view (no copy)."""
        addr = U.profile_status(self.profile)
        off = addr - self.ws.data_ptr()
        return self.ws[off:off + 4].view(torch.int32)

    def schedule(self, stream=None):
        U.schedule_batches(self.profile, self.cfg, self.order, self.offsets, self.num_batches, stream)

    def stats(self, stream=None):
        U.batch_stats(self.profile, self.cfg, self.offsets, self.num_batches, self.per_batch,
                      self.totals, stream)

    def simulate(self, arrival_us, stream=None, per_batch: bool = True, per_query: bool = True):
        """NEXT f2: sequential execution of the current schedule with arrivals (u64 us by caller
        index, torch int64/uint64 device tensor or numpy array).  Per-query latencies come back in
        scheduled order (latency[k] belongs to query order[k])."""
        if not hasattr(self, "sim_totals"):
            self.sim_totals = torch.zeros(U.SIM_TOTALS_BYTES, dtype=torch.uint8, device=self.device)
            self.batch_end = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.device)
            self.latency = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.device)
        U.simulate(self.profile, self.cfg, arrival_us, self.order, self.offsets, self.num_batches,
                   self.batch_end if per_batch else None, self.latency if per_query else None,
                   self.sim_totals, stream)

    def sim_results(self) -> dict:
        torch.cuda.synchronize(self.device)
        m = int(self.num_batches.item())
        tot = U.SimTotals.from_buffer_copy(self.sim_totals.cpu().numpy().tobytes())
        return {"batch_end": self.batch_end[:m].cpu().numpy().view(np.uint64),
                "latency": self.latency[: self.n].cpu().numpy().view(np.uint64),
                "totals": tot.as_dict()}

    def run(self, input_len, pred_out_len, slo_s, stream=None):
        self.load(input_len, pred_out_len, slo_s, stream)
        self.schedule(stream)
        self.stats(stream)

    def diagnostics(self, stream=None) -> dict:
        return U.get_diagnostics(self.profile, stream)

    # -- host views of the results (synchronising) -----------------------------------------
    def results(self) -> dict:
        torch.cuda.synchronize(self.device)
        m = int(self.num_batches.item())
        order = self.order[: self.n].cpu().numpy().view(np.uint32)
        offsets = self.offsets[: m + 1].cpu().numpy().view(np.uint32)
        tot = U.Totals.from_buffer_copy(self.totals.cpu().numpy().tobytes())
        out = {"order": order, "offsets": offsets, "m": m, "totals": tot.as_dict()}
        if self.per_batch is not None:
            out["per_batch"] = self.per_batch[:m].cpu().numpy().reshape(-1).view(U.BATCH_STAT_DTYPE)
        return out


def schedule_host(input_len: np.ndarray, pred_out_len: np.ndarray, slo_s: np.ndarray, cfg,
                  device=None, stream=None):
    """End-to-end call with HOST arrays: the library stages the inputs to the device and
    returns order / offsets / totals to host memory."""
    dev = torch.device(device or "cuda")
    c = U.make_config(cfg)
    n = int(input_len.shape[0])
    wsb = U.workspace_bytes(n, c)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    p = U.profile_load(n, input_len, pred_out_len, slo_s, c, ws, wsb, stream)
    order = np.empty(max(n, 1), np.uint32)
    offsets = np.empty(n + 1, np.uint32)
    nb = np.zeros(1, np.uint64)
    U.schedule_batches(p, c, order, offsets, nb, stream)
    tot = U.Totals()
    U.batch_stats(p, c, offsets, nb, None, C.addressof(tot), stream)
    m = int(nb[0])
    return order[:n], offsets[: m + 1], m, tot.as_dict()
