"""GPU parity of the sequential-execution simulator (NEXT f2, uellm_simulate) against the
oracle (O8) on the same seeded schedules and arrivals: batch ends, per-query latencies and every
integer total bit-exact; the four doubles within 1e-6 relative."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

SIM_INT = ["n", "batches", "makespan_us", "busy_us", "idle_us", "gen_tokens", "viol", "latency_max_us",
           "latency_sum_us"]
SIM_DBL = ["mean_latency_s", "slo_violation_rate", "utilization", "throughput_tok_s"]


def gpu_sim(inp, out, slo, cfg, arrival, host_arrival=False):
    from paper_2409_14961_b200.scheduler import GpuScheduler
    dev = torch.device("cuda:0")
    g = GpuScheduler(len(inp), cfg, device=dev, per_batch=True)
    g.run(torch.from_numpy(np.ascontiguousarray(inp).view(np.int32)).to(dev),
          torch.from_numpy(np.ascontiguousarray(out).view(np.int32)).to(dev),
          torch.from_numpy(np.ascontiguousarray(slo)).to(dev))
    arr = np.ascontiguousarray(arrival, np.uint64)
    g.simulate(arr if host_arrival else torch.from_numpy(arr.view(np.int64)).to(dev))
    r = g.results()
    r["sim"] = g.sim_results()
    return r


def assert_sim_parity(inp, out, slo, cfg, arrival, host_arrival=False, nthreads=8):
    r = gpu_sim(inp, out, slo, cfg, arrival, host_arrival)
    o_order, o_offs, o_m, _ = oracle.schedule(inp, out, slo, cfg, nthreads=nthreads)
    assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs)
    ends, lat, tot = oracle.simulate(inp, out, slo, cfg, o_order, o_offs, arrival)
    sim = r["sim"]
    assert np.array_equal(sim["batch_end"], ends), "batch_end"
    assert np.array_equal(sim["latency"], lat), "latency"
    st = sim["totals"]
    for f in SIM_INT:
        assert st[f] == tot[f], (f, st[f], tot[f])
    for f in SIM_DBL:
        assert st[f] == pytest.approx(tot[f], rel=1e-6, abs=0), f
    assert st["status"] == 0
    return r


@pytest.mark.parametrize("seed", range(0, 40, 4))
def test_sim_c1(seed):
    inp, out, slo, cfg = W.c1(seed, lam=10**6)
    assert_sim_parity(inp, out, slo, cfg, W.poisson_arrivals(16, seed, 3_000))


@pytest.mark.parametrize("pattern", ["rand", "ties", "identical", "descending"])
def test_sim_small_random(pattern):
    for seed in range(12):
        n = 1 + seed % 12
        inp, out, slo, cfg = W.random_small(seed * 7 + 3, n, pattern)
        arrival = W.random_arrivals(n, seed, [1, 100, 10_000, 10**6][seed % 4])
        assert_sim_parity(inp, out, slo, cfg, arrival)


@pytest.mark.parametrize("mode", [W.MODE_SEG_DP, W.MODE_FIFO, W.MODE_SLO_ODBS, W.MODE_SORT_ONLY])
def test_sim_c2_modes(mode):
    inp, out, slo, cfg = W.c2(5)
    cfg = cfg.replace(mode=mode, w1=1.0, w2=0.05, threshold=400.0)
    assert_sim_parity(inp, out, slo, cfg, W.poisson_arrivals(len(inp), 5, W.MEAN_GAP_US["c2"]))


def test_sim_c3_windows_poisson():
    inp, out, slo, cfg = W.c3(7, n=1_000_000)
    cfg = cfg.replace(window=100_000)
    assert_sim_parity(inp, out, slo, cfg, W.poisson_arrivals(len(inp), 7, W.MEAN_GAP_US["c3"]))


def test_sim_many_chunks_random_arrivals():
    # sort-only: one batch per query -> 2930 chunks of 1024 batches (several chunks per thread
    # of the carry scan); arrivals in random order
    inp, out, slo, cfg = W.c3(9, n=3_000_000)
    cfg = cfg.replace(mode=W.MODE_SORT_ONLY, window=250_000)
    assert_sim_parity(inp, out, slo, cfg, W.random_arrivals(len(inp), 9, 10**10))


def test_sim_zero_arrivals_equals_stats_completion():
    inp, out, slo, cfg = W.c2(6, n=8000)
    r = assert_sim_parity(inp, out, slo, cfg, np.zeros(8000, np.uint64))
    # all present at t = 0 on one window: the GPU stats' completion times and viol_seq
    assert np.array_equal(r["sim"]["batch_end"], r["per_batch"]["completion_us"])
    assert r["sim"]["totals"]["viol"] == r["totals"]["viol_seq"]


def test_sim_host_arrivals():
    inp, out, slo, cfg = W.c3(10, n=200_000)
    assert_sim_parity(inp, out, slo, cfg.replace(window=50_000),
                      W.poisson_arrivals(len(inp), 10, 21_000), host_arrival=True)


def test_sim_overflow_status():
    inp, out, slo, cfg = W.c2(11, n=100)
    arr = np.full(100, 2**63 - 5, np.uint64)
    r = gpu_sim(inp, out, slo, cfg, arr)
    assert r["sim"]["totals"]["status"] == 4
    with pytest.raises(oracle.OracleError):
        o = oracle.schedule(inp, out, slo, cfg)
        oracle.simulate(inp, out, slo, cfg, o[0], o[1], arr)


def test_sim_empty():
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    cfg = W.SchedConfig()
    g = GpuScheduler(0, cfg, device="cuda:0")
    e = torch.zeros(0, dtype=torch.int32, device="cuda:0")
    g.run(e, e, torch.zeros(0, dtype=torch.float32, device="cuda:0"))
    tot = U.SimTotals()
    U.simulate(g.profile, g.cfg, None, None, g.offsets, g.num_batches, None, None,
               __import__("ctypes").addressof(tot))
    d = tot.as_dict()
    assert d["n"] == 0 and d["makespan_us"] == 0 and d["status"] == 0 and d["throughput_tok_s"] == 0.0


@pytest.mark.slow
def test_sim_c4_full_size():
    """bench.py's configuration: 10^8 queries, 10^6-query windows, Poisson arrivals; the oracle
    re-runs the whole timeline (the simulator is a single sequential timeline: no sampling)."""
    inp, out, slo, cfg = W.c4(0)
    arrival = W.poisson_arrivals(len(inp), 0, W.MEAN_GAP_US["c4"])
    assert_sim_parity(inp, out, slo, cfg, arrival, nthreads=16)
