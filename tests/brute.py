"""Brute-force reference for tiny windows (n <= 12-16): enumerate ALL 2^(n-1) contiguous
segmentations of the SLO-sorted stream, evaluate the objective straight from its
definition with Python integers (no overflow, no pruning, no DP), and pick the optimum
with the R9 tie rule.  Independent of oracle/ (shares no code with it).

Objective (R7, R8, R14):
  sum over batches B of  est(B) + lambda * #{q in B : slo_us(q) < est(B)}
  est(B) = t_batch + t_iter*O + t_tok*b*O + t_prefill*b*s    (s = max input, O = max output)
Feasible batch: b == 1, or kv_bytes_per_elem*b*l*h*(s+O) <= kv_cap_bytes (cap 0 = none),
and b <= max_batch; with split_on_slo_change all members share one SLO value.
R9: among optimal segmentations take the one whose batch-start list, read right to left,
is lexicographically smallest.
"""
from __future__ import annotations

import numpy as np


def slo_us_ref(slo_s: float) -> int:
    """R12: round-half-even of the double product slo_s * 1e6 (Python floats are IEEE
    doubles; round() is half-to-even)."""
    return int(round(float(np.float32(slo_s)) * 1e6))


def sorted_order(inp, out, slo):
    n = len(inp)
    su = [slo_us_ref(s) for s in slo]
    return sorted(range(n), key=lambda k: (su[k], int(out[k]), k)), su


def batch_cost(cfg, members, inp, out, su):
    b = len(members)
    s = max(int(inp[k]) for k in members)
    O = max(int(out[k]) for k in members)
    if b > cfg.max_batch:
        return None
    if cfg.split_on_slo_change and len({su[k] for k in members}) > 1:
        return None
    if b > 1 and cfg.kv_cap_bytes and cfg.kv_bytes_per_elem * b * cfg.n_layers * cfg.hidden * (s + O) > cfg.kv_cap_bytes:
        return None
    est = cfg.t_batch_us + cfg.t_iter_us * O + cfg.t_tok_us * b * O + cfg.t_prefill_us * b * s
    viol = sum(1 for k in members if su[k] < est)
    return est + cfg.lambda_us * viol


def brute_segmentation(inp, out, slo, cfg):
    """-> (order, batch starts (ascending), optimal cost) for a single window."""
    order, su = sorted_order(inp, out, slo)
    n = len(order)
    if n == 0:
        return order, [], 0
    best = None
    for mask in range(1 << (n - 1)):
        starts = [0] + [k + 1 for k in range(n - 1) if mask >> k & 1]
        bounds = starts + [n]
        total = 0
        for a, z in zip(bounds[:-1], bounds[1:]):
            c = batch_cost(cfg, order[a:z], inp, out, su)
            if c is None:
                total = None
                break
            total += c
        if total is None:
            continue
        key = (total, starts[::-1])
        if best is None or key < best:
            best = key
    return order, best[1][::-1], best[0]
