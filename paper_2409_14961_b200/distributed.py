"""Multi-GPU sharding of the scheduling path: windows are independent (no batch
crosses a window, O1/R15), so rank r owns the contiguous window block
[floor(N_w*r/P), floor(N_w*(r+1)/P)) of ONE job and runs the whole path on its own GPU with no
data-path collective.  The one exchange step (a9) is a single all_gather of fixed-size per-rank
records written by the library (uellm_exchange_pack: the rank's uellm_totals followed by its
boundary bitmap); every rank then rebuilds the whole job's batch_offsets and exact totals on its
GPU (uellm_exchange_combine).

torch.distributed is plumbing here (NCCL over NVLink on B200 boxes, gloo in the CPU tests); this
module does no scheduling arithmetic: rank -> window-block bookkeeping and buffer marshalling only.
"""
from __future__ import annotations

import numpy as np
import torch

from . import uellm as U


def window_block(n_windows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous window block of `rank` (balanced to within one window)."""
    return (n_windows * rank) // world, (n_windows * (rank + 1)) // world


def query_range(n: int, window: int, world: int, rank: int) -> tuple[int, int]:
    """Arrival-index range [q0, q1) of the windows owned by `rank` (window 0 = whole stream)."""
    wl = window or n
    nwin = (n + wl - 1) // wl if n else 0
    w0, w1 = window_block(nwin, world, rank)
    return min(n, w0 * wl), min(n, w1 * wl)


def query_begins(n: int, window: int, world: int) -> list[int]:
    """query_begin of uellm_exchange_combine: world + 1 entries, rank r owns [qb[r], qb[r+1])."""
    return [query_range(n, window, world, r)[0] for r in range(world)] + [n]


class Exchange:
    """a9 buffers of one rank: its record, the gathered records and the combine outputs."""

    def __init__(self, n_total: int, window: int, world: int, rank: int, device):
        self.world, self.rank = world, rank
        self.qb = query_begins(n_total, window, world)
        self.q0, self.q1 = self.qb[rank], self.qb[rank + 1]
        self.n_total = n_total
        self.n_max = max(b - a for a, b in zip(self.qb[:-1], self.qb[1:])) if world else 0
        self.rec_bytes = U.exchange_bytes(self.n_max)
        dev = torch.device(device)
        self.record = torch.zeros(self.rec_bytes, dtype=torch.uint8, device=dev)
        self.gathered = torch.zeros(world * self.rec_bytes, dtype=torch.uint8, device=dev)
        self.ws_bytes = U.exchange_workspace_bytes(n_total, world)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.offsets = torch.empty(n_total + 1, dtype=torch.int32, device=dev)
        self.num_batches = torch.zeros(1, dtype=torch.int64, device=dev)
        self.totals = torch.zeros(U.TOTALS_BYTES, dtype=torch.uint8, device=dev)

    def pack(self, profile, cfg, totals_dev, stream=None):
        U.exchange_pack(profile, cfg, totals_dev, self.record, self.n_max, stream)

    def all_gather(self, group=None, backend: str = "nccl"):
        """ONE collective: all_gather_into_tensor (NCCL); gloo (CPU / test runs) takes the list form."""
        import torch.distributed as dist
        if backend == "nccl":
            dist.all_gather_into_tensor(self.gathered, self.record, group=group)
        else:
            dist.all_gather(list(self.gathered.view(self.world, -1).unbind(0)), self.record, group=group)

    def combine(self, stream=None):
        U.exchange_combine(self.gathered, self.world, self.n_max, self.qb, self.ws, self.ws_bytes, self.offsets,
                           self.num_batches, self.totals, stream)

    def results(self) -> dict:
        torch.cuda.synchronize(self.offsets.device)
        m = int(self.num_batches.item())
        tot = U.Totals.from_buffer_copy(self.totals.cpu().numpy().tobytes())
        return {"offsets": self.offsets[: m + 1].cpu().numpy().view(np.uint32), "m": m, "totals": tot.as_dict()}
