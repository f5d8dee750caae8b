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


def brute_simulate(inp, out, slo, cfg, order, offsets, arrival):
    """Discrete-event reference of the sequential-execution simulator (NEXT f2):
    one server, batches taken in plan order; a batch starts when the server is idle AND every
    member has arrived; its service time is est(B) (R7).  Formulated as an event loop
    over arrival / completion events with a heap (not as the max-plus recurrence the oracle
    and the GPU use).  Returns (batch_end list, latency dict by caller index, totals dict)."""
    import heapq
    n = len(inp)
    m = len(offsets) - 1
    members = [[int(order[k]) for k in range(int(offsets[t]), int(offsets[t + 1]))] for t in range(m)]
    batch_of = {x: t for t in range(m) for x in members[t]}
    missing = [len(ms) for ms in members]

    def est(ms):
        b = len(ms)
        s = max(int(inp[x]) for x in ms)
        O = max(int(out[x]) for x in ms)
        return cfg.t_batch_us + cfg.t_iter_us * O + cfg.t_tok_us * b * O + cfg.t_prefill_us * b * s

    ev = [(int(arrival[x]), 0, x) for x in range(n)]      # (time, kind 0 = arrival, query)
    heapq.heapify(ev)
    nxt, busy, ends, lat = 0, False, [None] * m, {}
    while ev:
        now = ev[0][0]
        while ev and ev[0][0] == now:                      # all events at this instant
            _, kind, x = heapq.heappop(ev)
            if kind == 0:
                missing[batch_of[x]] -= 1
            else:
                busy = False
                ends[x] = now
                for q in members[x]:
                    lat[q] = now - int(arrival[q])
            while not busy and nxt < m and missing[nxt] == 0:
                e = est(members[nxt])
                if e == 0:                                 # zero service time: done at once
                    ends[nxt] = now
                    for q in members[nxt]:
                        lat[q] = now - int(arrival[q])
                    nxt += 1
                    continue
                heapq.heappush(ev, (now + e, 1, nxt))
                busy = True
                nxt += 1
    assert nxt == m and all(e is not None for e in ends)
    su = [slo_us_ref(s) for s in slo]
    busy_us = sum(est(ms) for ms in members)
    mk = ends[-1] if m else 0
    tot = {"makespan_us": mk, "busy_us": busy_us, "idle_us": mk - busy_us,
           "gen_tokens": sum(len(ms) * max(int(out[x]) for x in ms) for ms in members),
           "viol": sum(1 for x in range(n) if lat[x] > su[x]),
           "latency_max_us": max(lat.values()) if n else 0,
           "latency_sum_us": sum(lat.values())}
    return ends, lat, tot
