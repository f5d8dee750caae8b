"""Pins of the oracle's sequential-execution simulator (oracle O8, NEXT f2) against things other
than itself (-m "not gpu"): an independent discrete-event simulator on small inputs (any
order, any partition), the SPEC worked example S:455, the all-at-t=0 special case that reduces
to the stats' completion times, and SPEC's invariants S:470-472."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.brute import brute_simulate, slo_us_ref


def random_plan(rng, n):
    order = rng.permutation(n).astype(np.uint32)
    cuts = sorted(rng.choice(np.arange(1, n), size=int(rng.integers(0, n)), replace=False).tolist()) if n > 1 else []
    return order, np.array([0] + cuts + [n], np.uint32)


@pytest.mark.parametrize("seed", range(40))
def test_simulate_vs_event_driven_brute(seed):
    # random queries, random (not scheduler-produced) order and partition, arrivals in any
    # order: the oracle's recurrence must agree with the event loop on every output
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 14))
    inp, out, slo, cfg = W.random_small(seed, n, ["rand", "ties", "identical"][seed % 3])
    order, offsets = random_plan(rng, n)
    hi = int(rng.choice([1, 50, 5_000, 500_000]))
    arrival = W.random_arrivals(n, seed, hi) if seed % 2 else W.poisson_arrivals(n, seed, hi / 4 + 1)
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, order, offsets, arrival)
    b_ends, b_lat, b_tot = brute_simulate(inp, out, slo, cfg, order, offsets, arrival)
    assert [int(e) for e in ends] == b_ends
    assert [int(x) for x in lat] == [b_lat[int(order[k])] for k in range(n)]
    for k in ("makespan_us", "busy_us", "idle_us", "gen_tokens", "viol", "latency_max_us", "latency_sum_us"):
        assert tot[k] == b_tot[k], k


@pytest.mark.parametrize("seed", range(6))
def test_simulate_seg_dp_schedule_vs_brute(seed):
    # the scheduler's own output as the plan (c1-shaped, BJ configs[0])
    inp, out, slo, cfg = W.c1(seed, lam=10**6)
    order, offsets, m, _ = oracle.schedule(inp, out, slo, cfg)
    arrival = W.poisson_arrivals(len(inp), seed, 3_000)
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, order, offsets, arrival)
    b_ends, b_lat, b_tot = brute_simulate(inp, out, slo, cfg, order, offsets, arrival)
    assert [int(e) for e in ends] == b_ends and tot["viol"] == b_tot["viol"]
    assert tot["latency_sum_us"] == b_tot["latency_sum_us"]


def test_spec_s455_single_request():
    # one request, one device hosting all layers, performance P, output n, zero comm
    # -> latency = n / P + 0 wait.  P = 50 tokens/s -> 20,000 us per token (R7: t_tok only),
    # n = 37 tokens -> 740,000 us, whatever the arrival time.
    cfg = W.SchedConfig(max_batch=1, t_batch_us=0, t_iter_us=0, t_tok_us=20_000, t_prefill_us=0)
    inp, out, slo = np.array([5], np.uint32), np.array([37], np.uint32), np.array([1.0], np.float32)
    for arr in (0, 123_456):
        ends, lat, tot = oracle.simulate(inp, out, slo, cfg, np.array([0], np.uint32),
                                         np.array([0, 1], np.uint32), np.array([arr], np.uint64))
        assert int(lat[0]) == 740_000 and int(ends[0]) == arr + 740_000
        assert tot["idle_us"] == arr and tot["busy_us"] == 740_000
        assert tot["viol"] == 0 and tot["gen_tokens"] == 37
    # S:451 "latency > slo": a latency equal to the SLO is met, one microsecond less is not
    for slo_s, v in ((0.74, 0), (0.739999, 1)):
        _, lat, tot = oracle.simulate(inp, out, np.array([slo_s], np.float32), cfg, np.array([0], np.uint32),
                                      np.array([0, 1], np.uint32), np.array([0], np.uint64))
        assert slo_us_ref(slo_s) in (740_000, 739_999) and int(lat[0]) == 740_000 and tot["viol"] == v


def test_spec_s457_empty():
    # empty plan list -> zero-throughput metrics
    cfg = W.SchedConfig()
    e = np.zeros(0, np.uint32)
    ends, lat, tot = oracle.simulate(e, e, np.zeros(0, np.float32), cfg, e, np.array([0], np.uint32),
                                     np.zeros(0, np.uint64))
    assert tot["makespan_us"] == 0 and tot["throughput_tok_s"] == 0.0 and tot["viol"] == 0


@pytest.mark.parametrize("gen", [lambda: W.c2(0, n=3000), lambda: W.c3(1, n=20_000)])
def test_all_present_at_zero_reduces_to_stats(gen):
    # arrivals all 0 on one window: the simulator's batch ends are the stats' completion
    # times (inclusive prefix of est), its latencies their per-batch values and its
    # violations viol_seq (slo_us < completion)
    inp, out, slo, cfg = gen()
    order, offsets, m, _ = oracle.schedule(inp, out, slo, cfg)
    pb, st = oracle.stats(inp, out, slo, cfg, order, offsets)
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, order, offsets, np.zeros(len(inp), np.uint64))
    assert np.array_equal(ends, pb["completion_us"])
    assert tot["viol"] == st["viol_seq"] and tot["idle_us"] == 0
    assert tot["makespan_us"] == st["makespan_us"]
    assert tot["latency_sum_us"] == int(np.sum(pb["size"].astype(object) * pb["completion_us"].astype(object)))
    assert tot["mean_latency_s"] == pytest.approx(st["mean_latency_s"], rel=1e-12)


def test_spread_arrivals_every_batch_waits():
    # gaps larger than any service time: every batch starts at its latest arrival
    inp, out, slo, cfg = W.c2(2, n=2000)
    order, offsets, m, _ = oracle.schedule(inp, out, slo, cfg)
    pb, _ = oracle.stats(inp, out, slo, cfg, order, offsets)
    arrival = np.zeros(len(inp), np.uint64)
    big = int(pb["est_us"].max()) + 1
    for t in range(m):                                   # batch t's members arrive at t*big ... t*big + 7
        mem = order[offsets[t]:offsets[t + 1]]
        arrival[mem] = t * big + np.arange(len(mem)) % 8
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, order, offsets, arrival)
    last = np.array([arrival[order[offsets[t]:offsets[t + 1]]].max() for t in range(m)], np.uint64)
    assert np.array_equal(ends, last + pb["est_us"])


@pytest.mark.parametrize("seed", range(3))
def test_invariants_s470_472(seed):
    inp, out, slo, cfg = W.c3(seed, n=30_000)
    cfg = cfg.replace(window=10_000)
    order, offsets, m, _ = oracle.schedule(inp, out, slo, cfg)
    pb, _ = oracle.stats(inp, out, slo, cfg, order, offsets)
    arrival = W.poisson_arrivals(len(inp), seed, 21_000)
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, order, offsets, arrival)
    est = pb["est_us"].astype(np.int64)
    start = ends.astype(np.int64) - est
    last = np.array([arrival[order[offsets[t]:offsets[t + 1]]].max() for t in range(m)], np.int64)
    prev = np.concatenate([[0], ends[:-1].astype(np.int64)])
    # work conservation: never start early, never idle without waiting for an arrival
    assert np.all(start >= prev) and np.all(start >= last)
    assert np.all((start == prev) | (start == last))
    assert tot["makespan_us"] == tot["busy_us"] + tot["idle_us"] and tot["busy_us"] == int(est.sum())
    # conservation: every query finishes once, after its arrival, no earlier than its batch's service
    bt = np.repeat(np.arange(m), np.diff(offsets.astype(np.int64)))
    assert np.array_equal(lat.astype(np.int64), ends[bt].astype(np.int64) - arrival[order].astype(np.int64))
    # metric consistency
    assert tot["throughput_tok_s"] * tot["makespan_us"] * 1e-6 == pytest.approx(tot["gen_tokens"], rel=1e-12)
    assert 0.0 < tot["utilization"] <= 1.0
    su = np.array([slo_us_ref(s) for s in slo[:2000]])
    lat_by_query = np.empty(len(inp), np.int64)
    lat_by_query[order] = lat.astype(np.int64)
    assert tot["viol"] >= int(np.sum(lat_by_query[:2000] > su))


def test_overflow_is_an_error():
    cfg = W.SchedConfig(max_batch=1)
    inp, out, slo = np.array([1], np.uint32), np.array([1], np.uint32), np.array([1.0], np.float32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.simulate(inp, out, slo, cfg, np.array([0], np.uint32), np.array([0, 1], np.uint32),
                        np.array([2**63 - 10], np.uint64))
    assert e.value.status == 4
