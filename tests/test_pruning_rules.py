"""The SEG-DP kernel's exact candidate pruning rules, checked as mathematics on the CPU (-m "not
gpu"): a plain sequential DP that drops candidates by D1 and by the penalty-aware D1' (DESIGN.md
section 7, a6 step 5) must reproduce the oracle's full-window DP (no pruning) -- every optimal
cost and every smallest-argmin breakpoint.  Pruning is evaluated at every boundary here (the
kernel prunes at block ends, a subset of these deaths), against every later live candidate."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.brute import slo_us_ref


def pruned_dp(inp, out, slo, cfg):
    order = sorted(range(len(inp)), key=lambda k: (slo_us_ref(slo[k]), int(out[k]), k))
    I = [int(inp[k]) for k in order]
    O = [int(out[k]) for k in order]
    S = [slo_us_ref(slo[k]) for k in order]
    n, Wm, lam = len(I), cfg.max_batch, cfg.lambda_us
    unit = cfg.kv_bytes_per_elem * cfg.n_layers * cfg.hidden
    cap = cfg.kv_cap_bytes // unit if cfg.kv_cap_bytes else None

    def est(i, j):
        b, s, o = j - i, max(I[i:j]), max(O[i:j])
        return cfg.t_batch_us + cfg.t_iter_us * o + cfg.t_tok_us * b * o + cfg.t_prefill_us * b * s

    def cost(i, j):
        e = est(i, j)
        return e + lam * sum(1 for k in range(i, j) if S[k] < e)

    def feasible(i, j):
        b = j - i
        return b == 1 or (b <= Wm and (cap is None or b * (max(I[i:j]) + max(O[i:j])) <= cap))

    C = [0] * (n + 1)
    arg = [0] * (n + 1)
    live = [0]
    for j in range(1, n + 1):
        live = [i for i in live if j - i <= Wm or j - i == 1]
        best = None
        for i in live:
            if not feasible(i, j):
                continue
            v = C[i] + cost(i, j)
            if best is None or v < best:
                best, arg[j] = v, i
        C[j] = best
        live.append(j)
        # prune at the state of boundary j (valid for every later boundary)
        keep = []
        for a, i in enumerate(live):
            dead = False
            for i2 in live[a + 1:]:
                mo, mi = max(O[i2:j]) if i2 < j else 0, max(I[i2:j]) if i2 < j else 0
                slope = cfg.t_tok_us * mo + cfg.t_prefill_us * mi
                rhs = (i2 - i) * slope
                one_run = len(set(S[i:j])) == 1 if i < j else True
                if lam and one_run and i2 < j and S[j - 1] < est(i2, j):
                    rhs += lam * (i2 - i)                       # D1'
                if C[i2] - C[i] < rhs:                          # D1 (+ D1')
                    dead = True
                    break
            if not dead:
                keep.append(i)
        live = keep
    return C[n], arg


@pytest.mark.parametrize("seed", range(40))
def test_pruned_dp_equals_full_dp(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 90))
    inp = rng.integers(1, 60, size=n).astype(np.uint32)
    out = (rng.integers(1, 20, size=n) * 8).astype(np.uint32)
    cls = np.array([0.002, 0.02, 0.2], np.float32) if seed % 2 else np.array([0.003], np.float32)
    slo = cls[rng.integers(0, len(cls), size=n)]
    cfg = W.SchedConfig(max_batch=int(rng.integers(4, 40)), lambda_us=int(rng.choice([10**6, 10**9, 37])),
                        t_batch_us=int(rng.integers(0, 500)), t_iter_us=int(rng.integers(1, 40)),
                        t_tok_us=int(rng.integers(0, 10)), t_prefill_us=int(rng.integers(0, 5)),
                        kv_cap_bytes=int(rng.choice([0, 4 * 32 * 4096 * 600])))
    c, arg = pruned_dp(inp, out, slo, cfg)
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp, out, slo, cfg)
    assert c == o_cost
    starts, j = [], n
    while j > 0:
        starts.append(arg[j])
        j = arg[j]
    assert sorted(starts) + [n] == [int(x) for x in o_offs]
