"""Multi-GPU sharding of the scheduling path: windows are independent (no batch
crosses a window, O1), so rank r owns the contiguous window block
[floor(N_w*r/P), floor(N_w*(r+1)/P)) and runs the whole path on its own GPU with no data-path
collective.  The one exchange step (a9) is a single all_gather of fixed-size per-rank totals.

torch.distributed is plumbing here (NCCL on GPUs, gloo in the CPU tests); no scheduling
arithmetic happens in this module.
"""
from __future__ import annotations

import numpy as np
import torch

TOTAL_FIELDS = ["n", "batches", "gen_tokens", "pad_in", "pad_out", "kv_bytes_max", "dp_cost",
                "viol_alone", "viol_seq", "over_cap", "makespan_us"]
GATHER_WORDS = 16          # 11 integer totals + 2 doubles (as raw bits) + 3 pad


def window_block(n_windows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous window block of `rank` (balanced to within one window)."""
    return (n_windows * rank) // world, (n_windows * (rank + 1)) // world


def query_range(n: int, window: int, world: int, rank: int) -> tuple[int, int]:
    """Arrival-index range [q0, q1) of the windows owned by `rank` (window 0 = whole stream)."""
    wl = window or n
    nwin = (n + wl - 1) // wl if n else 0
    w0, w1 = window_block(nwin, world, rank)
    return min(n, w0 * wl), min(n, w1 * wl)


def pack_totals(totals: dict, device) -> torch.Tensor:
    """Per-rank totals -> fixed-size int64 vector (doubles carried bit-exactly)."""
    v = np.zeros(GATHER_WORDS, np.int64)
    for k, f in enumerate(TOTAL_FIELDS):
        v[k] = np.int64(np.uint64(totals[f]).view(np.int64))
    v[11] = np.array([totals["mean_latency_s"]], np.float64).view(np.int64)[0]
    v[12] = np.array([totals["throughput_tok_s"]], np.float64).view(np.int64)[0]
    return torch.from_numpy(v).to(device)


def all_gather_totals(mine: torch.Tensor, group=None) -> torch.Tensor:
    """a9: one all_gather_into_tensor of the fixed-size per-rank buffers -> [world, 16]."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world * GATHER_WORDS, dtype=torch.int64, device=mine.device)
    dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    return out.view(world, GATHER_WORDS)


def combine_totals(gathered: torch.Tensor) -> dict:
    """Whole-job totals from the per-rank rows (sums; max for kv_bytes_max; the two means are
    re-weighted exactly from their integer numerators where possible)."""
    g = gathered.cpu().numpy()
    u = g[:, :11].view(np.uint64)
    out = {}
    for k, f in enumerate(TOTAL_FIELDS):
        col = [int(x) for x in u[:, k]]
        out[f] = max(col) if f == "kv_bytes_max" else sum(col)
    lat = g[:, 11].view(np.float64)
    ns = [int(x) for x in u[:, 0]]
    n = sum(ns)
    out["mean_latency_s"] = float(sum(l * m for l, m in zip(lat, ns)) / n) if n else 0.0
    mk = out["makespan_us"]
    out["throughput_tok_s"] = out["gen_tokens"] / (mk * 1e-6) if mk else 0.0
    return out
