"""Pins of the CPU oracle against things other than itself (-m "not gpu"):
brute force on tiny inputs, closed forms, special cases, SPEC worked examples
and invariants.  Each test cites the passage it checks."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from tests.brute import brute_segmentation, slo_us_ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sizes_of(offsets):
    return list(np.diff(np.asarray(offsets, np.int64)))


# ---------------------------------------------------------------- O2 slo_us (R12)
@pytest.mark.parametrize("x,us", [
    (0.5, 500_000),                 # exact
    (1.0 / 128, 7812),              # 7812.5 exactly -> half-to-even -> 7812
    (3.0 / 128, 23438),             # 23437.5 exactly -> half-to-even -> 23438
    (5.0 / 128, 39062),             # 39062.5 -> 39062
    (350.0, 350_000_000),           # P:463 upper end
    (1.0, 1_000_000),               # P:463 lower end
    (4294.0, 4_294_000_000),
])
def test_slo_us_closed_form(x, us):
    assert oracle.slo_us(x) == us


@pytest.mark.parametrize("x", [0.0, -1.0, float("inf"), float("nan"), 4.0e-7, 4296.0])
def test_slo_us_contract(x):
    # S:266 / S:98: invalid SLO is a typed rejection; 4e-7 s rounds to 0 us; 4296 s > 2^32-1 us
    with pytest.raises(oracle.OracleError) as e:
        oracle.slo_us(x)
    assert e.value.status == 2


# ---------------------------------------------------------------- A1 KV bytes
def test_kv_bytes_spec_examples():
    assert oracle.kv_bytes(4, 1, 1, 1, 0, 1) == 4                     # S:134 [PAPER]
    assert oracle.kv_bytes(4, 1, 1, 1, 0, 0) == 0                     # S:135 [TRIVIAL]
    assert oracle.kv_bytes(4, 8, 32, 4096, 512, 512) == 4_294_967_296  # S:136 [DERIVED]
    with pytest.raises(oracle.OracleError) as e:
        oracle.kv_bytes(4, 2**40, 32, 4096, 2**20, 2**20)
    assert e.value.status == 4                                         # S:133 sizing error


def test_kv_bytes_monotone():
    # nondecreasing in every argument
    base = (4, 3, 5, 7, 11, 13)
    v0 = oracle.kv_bytes(*base)
    for k in range(6):
        a = list(base); a[k] += 1
        assert oracle.kv_bytes(*a) >= v0


# ---------------------------------------------------------------- O7 token accounting
def _stats_of(inp, out, slo, groups, cfg=None):
    cfg = cfg or W.SchedConfig(mode=W.MODE_FIFO, max_batch=64)
    order = np.array([k for g in groups for k in g], np.uint32)
    offs = np.cumsum([0] + [len(g) for g in groups]).astype(np.uint32)
    return oracle.stats(np.asarray(inp), np.asarray(out), np.asarray(slo, np.float32), cfg, order, offs)


def test_batch_token_cost_spec_examples():
    pb, _ = _stats_of([10], [20], [1.0], [[0]])
    assert (pb["gen_tokens"][0], pb["pad_in"][0]) == (20, 0)
    pb, _ = _stats_of([10, 30], [5, 50], [1.0, 1.0], [[0, 1]])
    assert (pb["gen_tokens"][0], pb["pad_in"][0]) == (100, 20)
    pb, _ = _stats_of([7, 7, 7], [9, 9, 9], [1.0] * 3, [[0, 1, 2]])
    assert (pb["gen_tokens"][0], pb["pad_in"][0]) == (27, 0)


def test_plan_token_cost_spec_example():
    inp, out, slo = [1, 1, 1, 1], [5, 5, 50, 50], [1.0] * 4
    _, split = _stats_of(inp, out, slo, [[0, 1], [2, 3]])
    _, single = _stats_of(inp, out, slo, [[0, 1, 2, 3]])
    assert split["gen_tokens"] == 110 and single["gen_tokens"] == 200


def test_fig3_structural_claim():
    # P:210 / Fig. 3: splitting by output length needs fewer generated tokens and paddings
    # than one default batch (lengths lost -> structural pin only).
    inp, out, slo = [8, 10, 12], [50, 10, 8], [1.0] * 3
    _, one = _stats_of(inp, out, slo, [[0, 1, 2]])
    _, two = _stats_of(inp, out, slo, [[0], [1, 2]])
    assert two["gen_tokens"] < one["gen_tokens"] and two["pad_in"] < one["pad_in"]


def test_stats_completion_and_violations():
    # sequential execution; completion = prefix sum of est; viol_seq >= viol_alone
    cfg = W.SchedConfig(mode=W.MODE_FIFO, max_batch=2, t_batch_us=10, t_iter_us=1,
                        t_tok_us=1, t_prefill_us=1)
    inp, out, slo = [1, 2, 3], [4, 5, 6], [25e-6, 60e-6, 40e-6]
    pb, tot = _stats_of(inp, out, slo, [[0, 1], [2]], cfg)
    e0 = 10 + 1 * 5 + 1 * 2 * 5 + 1 * 2 * 2       # 29
    e1 = 10 + 6 + 6 + 3                           # 25
    assert list(pb["est_us"]) == [e0, e1]
    assert list(pb["completion_us"]) == [e0, e0 + e1]
    assert list(pb["viol_alone"]) == [1, 0]       # 25 < 29, 60 >= 29 ; 40 >= 25
    assert list(pb["viol_seq"]) == [1, 1]         # completion 29 ; 40 < 54 = 29 + 25
    assert tot["makespan_us"] == e0 + e1
    assert tot["mean_latency_s"] == pytest.approx((2 * e0 + (e0 + e1)) / 3 * 1e-6, rel=1e-15)
    assert tot["throughput_tok_s"] == pytest.approx((2 * 5 + 6) / ((e0 + e1) * 1e-6), rel=1e-15)


# ---------------------------------------------------------------- O4 SEG-DP vs brute force
PATTERNS = ["rand", "ties", "bucket", "identical", "descending", "classes"]


@pytest.mark.parametrize("pattern", PATTERNS)
def test_segdp_equals_brute_force(pattern):
    for seed in range(120):
        n = 1 + seed % 10
        inp, out, slo, cfg = W.random_small(seed * 7 + 1, n, pattern)
        order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
        b_order, b_starts, b_cost = brute_segmentation(inp, out, slo, cfg)
        assert list(order) == b_order, (seed, pattern)
        assert cost == b_cost, (seed, pattern, cfg)
        assert list(offs[:-1]) == b_starts, (seed, pattern, cfg)
        _, tot = oracle.stats(inp, out, slo, cfg, order, offs)
        assert tot["dp_cost"] == cost


@pytest.mark.parametrize("seed", range(6))
def test_segdp_c1_brute_force(seed):
    # BJ configs[0]: 16 queries, brute-force checkable (2^15 segmentations)
    for lam in (0, 10**6):
        inp, out, slo, cfg = W.c1(seed, lam)
        order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
        b_order, b_starts, b_cost = brute_segmentation(inp, out, slo, cfg)
        assert (list(order), list(offs[:-1]), cost) == (b_order, b_starts, b_cost)


@pytest.mark.parametrize("n,w,sizes", [(10, 4, [2, 4, 4]), (37, 8, [5, 8, 8, 8, 8]),
                                       (16, 16, [16]), (17, 16, [1, 16])])
def test_segdp_identical_closed_form(n, w, sizes):
    # identical queries, lambda = 0, no binding cap, t_batch + t_iter*o > 0:
    # k = ceil(n/W) batches, the first is the remainder (R9 tie rule)
    cfg = W.SchedConfig(max_batch=w, lambda_us=0)
    inp = np.full(n, 100, np.uint32); out = np.full(n, 200, np.uint32)
    slo = np.full(n, 10.0, np.float32)
    _, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    assert sizes_of(offs) == sizes
    per_q = cfg.t_tok_us * 200 + cfg.t_prefill_us * 100
    assert cost == len(sizes) * (cfg.t_batch_us + cfg.t_iter_us * 200) + n * per_q


def test_segdp_w1_singletons():
    inp, out, slo, cfg = W.c2(0, n=500)
    _, offs, m, _ = oracle.schedule(inp, out, slo, cfg.replace(max_batch=1))
    assert m == 500 and sizes_of(offs) == [1] * 500


def test_segdp_zero_overhead_merges_only_zero_padding():
    # t_batch = t_iter = lambda = 0: batching never pays, ties prefer merging, so every
    # batch has zero padding and the cost is the constant useful work (SURVEY 8(c) O4 special)
    inp, out, slo, cfg = W.c2(3, n=400)
    inp = (inp % 3 + 1).astype(np.uint32); out = (out % 2 + 1).astype(np.uint32)
    cfg = cfg.replace(t_batch_us=0, t_iter_us=0, lambda_us=0)
    order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    pb, tot = oracle.stats(inp, out, slo, cfg, order, offs)
    assert tot["pad_in"] == 0 and tot["pad_out"] == 0
    assert cost == cfg.t_tok_us * int(out.sum()) + cfg.t_prefill_us * int(inp.sum())


def test_segdp_all_violating_equals_lambda0():
    # every batch violates all members (slo 1 ms < t_batch + t_iter): the penalty is a
    # constant lambda*n, so the segmentation equals the lambda = 0 one (c5-ii)
    inp, out, _, cfg = W.c3(1, n=3000)
    slo = np.full(3000, 1e-3, np.float32)
    _, offs_a, _, cost_a = oracle.schedule(inp, out, slo, cfg.replace(lambda_us=10**9))
    _, offs_b, _, cost_b = oracle.schedule(inp, out, slo, cfg.replace(lambda_us=0))
    assert np.array_equal(offs_a, offs_b)
    assert cost_a == cost_b + 10**9 * 3000


# ---------------------------------------------------------------- invariants at scale
def _check_invariants(inp, out, slo, cfg, order, offs):
    n = len(inp)
    # partition: every query exactly once
    assert sorted(order.tolist()) == list(range(n))
    assert offs[0] == 0 and offs[-1] == n and np.all(np.diff(offs.astype(np.int64)) > 0)
    # SLO ordering preserved (BJ): scan order is (slo_us, out, idx) ascending
    su = np.array([slo_us_ref(s) for s in slo[order]], np.int64)
    if cfg.mode != W.MODE_FIFO:
        key = su * 2**33 + out[order].astype(np.int64) * 2**0
        assert np.all(np.diff(key) >= 0)
    pb, tot = oracle.stats(inp, out, slo, cfg, order, offs)
    assert int(pb["size"].sum()) == n
    assert np.all(pb["size"] <= cfg.max_batch)
    # memory cap respected unless a query alone exceeds it (R10)
    if cfg.kv_cap_bytes:
        assert np.all((pb["kv_bytes"] <= cfg.kv_cap_bytes) | (pb["size"] == 1))
    assert np.all(pb["viol_seq"] >= pb["viol_alone"])
    assert np.all(pb["gen_tokens"] == pb["size"].astype(np.uint64) * pb["max_out"])
    return pb, tot


@pytest.mark.parametrize("gen,kw", [(W.c2, dict(n=3000)), (W.c2, dict(n=3000, split=1)),
                                    (W.c3, dict(n=20000)), (W.c3, dict(n=20000, lam=0))])
def test_segdp_upper_bounds_and_invariants(gen, kw):
    inp, out, slo, cfg = gen(11, **kw)
    order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    pb, tot = _check_invariants(inp, out, slo, cfg, order, offs)
    assert tot["dp_cost"] == cost
    # C_DP <= cost of any feasible segmentation: all singletons, Alg. 1, FIFO-on-sorted chunks
    for mode, extra in ((W.MODE_SORT_ONLY, {}), (W.MODE_SLO_ODBS, dict(w1=1.0, w2=0.01, threshold=500.0))):
        c2 = cfg.replace(mode=mode, **extra)
        o2, f2, _, _ = oracle.schedule(inp, out, slo, c2)
        _check_invariants(inp, out, slo, c2, o2, f2)
        _, t2 = oracle.stats(inp, out, slo, cfg, o2, f2)
        assert cost <= t2["dp_cost"]


def test_windows_are_independent():
    # O1: windows are consecutive chunks of the arrival stream; no batch crosses one
    inp, out, slo, cfg = W.c3(5, n=5000)
    cfg = cfg.replace(window=1200)
    order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    tot_cost = 0
    for w0 in range(0, 5000, 1200):
        w1 = min(5000, w0 + 1200)
        o, f, _, c = oracle.schedule(inp[w0:w1], out[w0:w1], slo[w0:w1], cfg.replace(window=0))
        assert np.array_equal(order[w0:w1], o + w0)
        assert set((f + w0).tolist()) <= set(offs.tolist())
        tot_cost += c
    assert tot_cost == cost


def test_contract_error_on_invalid_query():
    inp, out, slo, cfg = W.c2(0, n=50)
    bad = inp.copy(); bad[7] = 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.schedule(bad, out, slo, cfg)
    assert e.value.status == 2
    s2 = slo.copy(); s2[3] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.schedule(inp, out, s2, cfg)


def test_empty_input():
    z = np.zeros(0, np.uint32)
    order, offs, m, cost = oracle.schedule(z, z, np.zeros(0, np.float32), W.SchedConfig())
    assert m == 0 and cost == 0 and list(offs) == [0]


# ---------------------------------------------------------------- O5 Alg. 1
def _alg1(inp, out, slo, **kw):
    cfg = W.SchedConfig(mode=W.MODE_SLO_ODBS, **kw)
    order, offs, m, _ = oracle.schedule(np.asarray(inp, np.uint32), np.asarray(out, np.uint32),
                                        np.asarray(slo, np.float32), cfg)
    return order.tolist(), [order[a:z].tolist() for a, z in zip(offs[:-1], offs[1:])]


def test_alg1_singleton():
    _, b = _alg1([5], [7], [3.0], threshold=1.0)
    assert b == [[0]]


def test_alg1_sorts_by_slo():
    order, _ = _alg1([1, 1, 1], [10, 10, 10], [300.0, 10.0, 100.0])  # S:269 P:256
    assert order == [1, 2, 0]


def test_alg1_latency_example():
    # w1=1, w2=0, L1=1, Threshold=100; (slo, len) = (10,.), (20,.), (90,.):
    # (20+10)*2*1 = 60 <= 100 admits r2; (90+20)*3 = 330 > 100 splits.  Holds for lengths
    # <= 50 (dynamic cap floor(100/len) >= 2; SURVEY 4.1 caveat).
    _, b = _alg1([1, 1, 1], [50, 40, 30], [10.0, 20.0, 90.0], w1=1.0, w2=0.0, l1=1.0,
                 threshold=100.0, max_batch=8)
    assert b == [[0, 1], [2]]
    # at length 51 the dynamic cap floor(100/51) = 1 flushes every query
    _, b = _alg1([1, 1, 1], [51, 51, 51], [10.0, 20.0, 90.0], w1=1.0, w2=0.0, threshold=100.0,
                 max_batch=8)
    assert b == [[0], [1], [2]]


def test_alg1_length_example():
    # w1=0 (SLO-DBS), w2=1, L2=1, Threshold=50, lengths {30, 25}:
    # T_o = (25-30)*2*1 = -10 <= 50 -> same batch (needs CM = w2*SLO <= 25)
    _, b = _alg1([1, 1], [30, 25], [5.0, 6.0], w1=0.0, w2=1.0, l2=1.0, threshold=50.0)
    assert b == [[0, 1]]
    # Eq. 2's additive form (R2): T_o = (25+30)*2 = 110 > 50 -> split
    _, b = _alg1([1, 1], [30, 25], [5.0, 6.0], w1=0.0, w2=1.0, threshold=50.0, eq2_additive=1)
    assert b == [[0], [1]]


@pytest.mark.parametrize("l1,expect", [(1.0, [[0, 1], [2]]), (2.0, [[0], [1], [2]]),
                                       (0.25, [[0, 1, 2]])])
def test_alg1_l1_scale(l1, expect):
    """Alg. 1 line 6: T_l = (q.SLO + L_CM) x (len(batch_c) + 1) x L1, worked by hand.
    w1 = 1, w2 = 0, Threshold = 100, (SLO, length) = (10, 30), (20, 30), (90, 30); the line-20 cap
    is floor(100 / CM) = floor(100 / 30) = 3 (R5):
      L1 = 1   : x=1 (20+10)*2*1 = 60 <= 100 admit; x=2 (90+20)*3*1 = 330 > 100 split
      L1 = 2   : x=1 (20+10)*2*2 = 120 > 100 split; x=2 (90+20)*2*2 = 440 > 100 split
      L1 = 0.25: x=1 15 <= 100 admit; x=2 (90+20)*3*0.25 = 82.5 <= 100 admit, |batch| = 3 = cap
    A misplaced L1 ((q.SLO*L1 + L_CM)*2 = 100 at L1 = 2 admits) or a dropped L1 fails."""
    _, b = _alg1([1, 1, 1], [30, 30, 30], [10.0, 20.0, 90.0], w1=1.0, w2=0.0, l1=l1,
                 threshold=100.0, max_batch=8)
    assert b == expect


@pytest.mark.parametrize("l2,lens,thr,expect", [
    (2.0, [10, 13, 13], 10.0, [[0], [1, 2]]),      # x=1: (13-10)*2*2 = 12 > 10 split
    (1.0, [10, 13, 13], 10.0, [[0, 1, 2]]),        # x=1: 6 <= 10; x=2: (13-13)*3 = 0
    (0.5, [10, 13, 13], 2.0, [[0], [1, 2]]),       # x=1: 3*2*0.5 = 3 > 2 split
    (0.1, [10, 10, 13], 0.9, [[0, 1, 2]]),         # x=2: ((13-10)*3)*0.1 = 0.9 <= 0.9 (binary64)
])
def test_alg1_l2_scale(l2, lens, thr, expect):
    """Alg. 1 line 7: T_o = (q.length - O_CM) x (len(batch_c) + 1) x L2, evaluated left to
    right as printed.  w1 = 0, w2 = 1 (SLO-DBS weights), SLO 0.1 s for all, so CM = 0.1 and
    the line-20 cap is floor(thr / 0.1) >= 3.  The last case pins the printed evaluation order:
    in binary64 (3*3)*0.1 == 0.9 but (3*0.1)*3 == 0.9000000000000001 > 0.9, so applying L2 before
    the (len(batch_c) + 1) factor splits the batch."""
    assert (3 * 3) * 0.1 == 0.9 and (3 * 0.1) * 3 > 0.9        # the arithmetic the case relies on
    _, b = _alg1([1, 1, 1], lens, [0.1, 0.1, 0.1], w1=0.0, w2=1.0, l2=l2, threshold=thr, max_batch=8)
    assert b == expect


@pytest.mark.parametrize("inp,cap,expect", [
    ([10, 10, 10, 10, 10], 160, [[0, 1], [2, 3], [4]]),   # kv(b) = 4*b*1*1*(10+10) = 80 b <= 160
    ([10, 10, 10, 10, 10], 159, [[0], [1], [2], [3], [4]]),
    ([10, 10, 10, 10, 10], 40, [[0], [1], [2], [3], [4]]),  # a query alone over the cap (R10)
    ([10, 50, 10], 400, [[0], [1], [2]]),                 # {0,1}: 4*2*(50+10) = 480 > 400;
                                                          # {1,2}: 4*2*(max(50,10)+10) = 480 > 400
    ([10, 50, 10], 480, [[0, 1], [2]]),                   # {0,1}: 480 <= 480 admit;
                                                          # {0,1,2}: 4*3*(50+10) = 720 > 480
])
def test_alg1_kv_cap_admission(inp, cap, expect):
    """R18: Alg. 1 has no memory test; a non-empty batch admits q only if its KV bytes
    4*b*l*h*(s + O) (s = max input, O = max output incl. q) stay <= the reserve.
    l = h = 1, kv_bytes_per_elem = 4, every output 10, SLO 1 s, w1 = 0, w2 = 1, threshold 1000
    (line-20 cap min(floor(1000/1), W = 8) = 8, T_o = 0): only the KV test splits."""
    _, b = _alg1(inp, [10] * len(inp), [1.0] * len(inp), w1=0.0, w2=1.0, threshold=1000.0,
                 max_batch=8, kv_bytes_per_elem=4, n_layers=1, hidden=1, kv_cap_bytes=cap)
    assert b == expect


def test_stats_pad_out_kv_over_cap_hand_values():
    """O7 hand values (S:144-146 extended to the output side and the KV cap):
    batch {(in 10, out 5), (in 30, out 50)}: pad_out = 2*50 - (5+50) = 45, pad_in = 2*30 - 40 = 20,
    kv = 4 * 2 * 32 * 4096 * (30 + 50) = 83,886,080 B; over_cap is strict (kv > cap)."""
    kv = 83_886_080
    for cap, oc in ((kv, 0), (kv - 1, 1), (0, 0)):
        cfg = W.SchedConfig(mode=W.MODE_FIFO, max_batch=64, kv_cap_bytes=cap)
        pb, tot = _stats_of([10, 30], [5, 50], [1.0, 1.0], [[0, 1]], cfg)
        assert (pb["pad_out"][0], pb["pad_in"][0], pb["kv_bytes"][0]) == (45, 20, kv)
        assert pb["over_cap"][0] == oc and tot["over_cap"] == oc
        assert (tot["pad_out"], tot["kv_bytes_max"]) == (45, kv)
    # two singletons: kv = 4*32*4096*30 = 15,728,640 and 4*32*4096*80 = 41,943,040 -> max; a single
    # query over the cap is admitted but counted (R10)
    cfg = W.SchedConfig(mode=W.MODE_FIFO, max_batch=64, kv_cap_bytes=20_000_000)
    pb, tot = _stats_of([10, 30], [20, 50], [1.0, 1.0], [[0], [1]], cfg)
    assert list(pb["kv_bytes"]) == [15_728_640, 41_943_040] and tot["kv_bytes_max"] == 41_943_040
    assert list(pb["over_cap"]) == [0, 1] and tot["over_cap"] == 1
    assert list(pb["pad_out"]) == [0, 0] and tot["pad_out"] == 0


def test_alg1_identical_requests_dynamic_cap():
    # identical requests form batches of the dynamic cap floor(thr/CM) (R5)
    _, b = _alg1([3] * 10, [9] * 10, [5.0] * 10, w1=0.0, w2=1.0, threshold=50.0, max_batch=64)
    assert [len(x) for x in b] == [10]
    _, b = _alg1([3] * 10, [9] * 10, [20.0] * 10, w1=0.0, w2=1.0, threshold=50.0, max_batch=64)
    assert [len(x) for x in b] == [2] * 5
    _, b = _alg1([3] * 10, [9] * 10, [5.0] * 10, w1=0.0, w2=1.0, threshold=50.0, max_batch=4)
    assert [len(x) for x in b] == [4, 4, 2]


def test_alg1_invariants_random():
    for seed in range(30):
        inp, out, slo, cfg = W.c2(seed, n=700, split=seed % 2)
        cfg = cfg.replace(mode=W.MODE_SLO_ODBS, w1=float(seed % 3), w2=0.5 * (seed % 2),
                          threshold=200.0 + 50 * seed)
        if cfg.w1 + cfg.w2 == 0:
            cfg = cfg.replace(w1=1.0)
        order, offs, m, _ = oracle.schedule(inp, out, slo, cfg)
        _check_invariants(inp, out, slo, cfg, order, offs)
        # per-batch minimum SLOs nondecreasing
        su = np.array([slo_us_ref(s) for s in slo[order]])
        mins = [su[a:z].min() for a, z in zip(offs[:-1], offs[1:])]
        assert all(x <= y for x, y in zip(mins, mins[1:]))


# ---------------------------------------------------------------- O6 FIFO
@pytest.mark.parametrize("n,cap,sizes", [(5, 2, [2, 2, 1]), (5, 9, [5]), (4, 1, [1, 1, 1, 1])])
def test_fifo(n, cap, sizes):
    cfg = W.SchedConfig(mode=W.MODE_FIFO, max_batch=cap)
    rng = np.random.default_rng(n)
    slo = rng.uniform(1, 9, n).astype(np.float32)
    order, offs, m, _ = oracle.schedule(np.ones(n, np.uint32), np.ones(n, np.uint32), slo, cfg)
    assert order.tolist() == list(range(n)) and sizes_of(offs) == sizes


# ---------------------------------------------------------------- committed goldens
def test_goldens():
    """tests/golden/*.json: small cases whose expected values come from the paper / SPEC
    (cited inside each file) or from brute force (tests/brute.py), never from the GPU."""
    files = sorted(f for f in os.listdir(GOLDEN) if f.endswith(".json"))
    assert files
    for f in files:
        g = json.load(open(os.path.join(GOLDEN, f)))
        cfg = W.SchedConfig(**g["config"])
        inp = np.array(g["input_len"], np.uint32); out = np.array(g["pred_out_len"], np.uint32)
        slo = np.array(g["slo_s"], np.float32)
        order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
        assert order.tolist() == g["order"], f
        assert offs.tolist() == g["offsets"], f
        if "dp_cost" in g:
            assert cost == g["dp_cost"], f
