"""Test-side reference of the a9 exchange record (include/uellm.h, uellm_exchange_*): plain numpy,
written from the header's description, independent of the library.  Used by the gloo tests on CPU
(ranks run the CPU oracle) and to cross-check the library's combine on the GPU.

record = [uellm_totals: 11 u64 (n .. makespan_us), 2 f64 (mean latency, throughput),
          latency_sum_lo, latency_sum_hi, overflow | u32 bitmap words of the rank's n_r + 1 bits],
padded to a 16-byte multiple with one spare bitmap word.
"""
from __future__ import annotations

import numpy as np

TOTAL_FIELDS = ["n", "batches", "gen_tokens", "pad_in", "pad_out", "kv_bytes_max", "dp_cost",
                "viol_alone", "viol_seq", "over_cap", "makespan_us"]


def record_bytes(n_max: int) -> int:
    b = 128 + 4 * ((n_max + 1 + 31) // 32 + 1)
    return (b + 15) // 16 * 16


def make_record(totals: dict, latency_sum: int, offsets_local, n_r: int, n_max: int) -> np.ndarray:
    """One rank's record from its totals (oracle dict), exact latency numerator and local offsets."""
    rec = np.zeros(record_bytes(n_max), np.uint8)
    w = np.zeros(16, np.uint64)
    for k, f in enumerate(TOTAL_FIELDS):
        w[k] = np.uint64(totals[f])
    w[11] = np.array([totals["mean_latency_s"]], np.float64).view(np.uint64)[0]
    w[12] = np.array([totals["throughput_tok_s"]], np.float64).view(np.uint64)[0]
    w[13] = np.uint64(latency_sum & (2**64 - 1))
    w[14] = np.uint64(latency_sum >> 64)
    rec[:128] = w.view(np.uint8)
    bits = np.zeros(n_r + 1, np.uint8)
    bits[np.asarray(offsets_local, np.int64)] = 1
    packed = np.packbits(bits, bitorder="little")
    rec[128:128 + len(packed)] = packed
    return rec


def combine(gathered: np.ndarray, query_begin) -> tuple[np.ndarray, dict]:
    """-> (job batch_offsets int64, job totals dict) from [world, record_bytes] uint8 records."""
    world = gathered.shape[0]
    tot = {f: 0 for f in TOTAL_FIELDS}
    lat = 0
    parts = []
    for r in range(world):
        w = gathered[r, :128].view(np.uint64)
        for k, f in enumerate(TOTAL_FIELDS):
            tot[f] = max(tot[f], int(w[k])) if f == "kv_bytes_max" else tot[f] + int(w[k])
        lat += int(w[13]) + (int(w[14]) << 64)
        q0, q1 = query_begin[r], query_begin[r + 1]
        bits = np.unpackbits(gathered[r, 128:], bitorder="little")[: q1 - q0]
        parts.append(np.flatnonzero(bits).astype(np.int64) + q0)
    offs = np.concatenate(parts + [np.array([query_begin[-1]], np.int64)])
    n = tot["n"]
    tot["latency_sum_us"] = lat
    tot["mean_latency_s"] = lat / n * 1e-6 if n else 0.0
    tot["throughput_tok_s"] = tot["gen_tokens"] / (tot["makespan_us"] * 1e-6) if tot["makespan_us"] else 0.0
    return offs, tot
