"""Multi-GPU sharding of the scheduling path: windows are independent (no batch
crosses a window, O1), so rank r owns the contiguous window block
[floor(N_w*r/P), floor(N_w*(r+1)/P)) and runs the whole path on its own GPU with no data-path
collective.  The one exchange step (a9) is a single all_gather of a fixed-size per-rank buffer:
the rank's totals (16 int64 words) followed by its boundary bitmap over its own scheduled
positions (uellm_boundary_bitmap: bit k set iff a batch starts at local position k, k = 0..n_r),
padded to the largest rank.  Every rank can then rebuild the whole job's batch_offsets.

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


def exchange_words(n_max: int) -> int:
    """int64 words of one rank's a9 buffer: totals + bitmap of n_max + 1 bits (u32 words, 2 per int64)."""
    u32 = (n_max + 1 + 31) // 32
    return GATHER_WORDS + (u32 + 1) // 2


def bitmap_view(buf: torch.Tensor) -> torch.Tensor:
    """The u32 bitmap region of one rank's int64 exchange buffer (a view: the library writes it in place)."""
    return buf[GATHER_WORDS:].view(torch.int32)


def all_gather_exchange(mine: torch.Tensor, group=None) -> torch.Tensor:
    """a9: ONE all_gather_into_tensor of the per-rank [totals | bitmap] buffers -> [world, words]."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world * mine.numel(), dtype=torch.int64, device=mine.device)
    dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    return out.view(world, mine.numel())


def global_offsets(gathered: torch.Tensor, ranges) -> np.ndarray:
    """Whole-job batch_offsets from the gathered buffers: rank r's set bits k (0 <= k <= n_r) are
    global positions q0_r + k; consecutive ranks share the boundary q1_r = q0_{r+1}."""
    g = gathered.cpu().numpy()
    parts = []
    for r, (q0, q1) in enumerate(ranges):
        n_r = q1 - q0
        words = g[r, GATHER_WORDS:].view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: n_r + 1]
        parts.append(np.flatnonzero(bits).astype(np.int64) + q0)
    allpos = np.concatenate(parts) if parts else np.zeros(1, np.int64)
    return np.unique(allpos)
