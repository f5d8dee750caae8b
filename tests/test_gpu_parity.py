"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle on the same seeded
inputs.  Bit-exact: order, batch_offsets, num_batches, dp_cost and every integer statistic;
mean_latency_s / throughput_tok_s within 1e-6 relative (north_star / SURVEY 8(c))."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

INT_FIELDS = ["start", "size", "max_in", "max_out", "gen_tokens", "pad_in", "pad_out", "kv_bytes",
              "est_us", "completion_us", "viol_alone", "viol_seq", "over_cap", "window"]
TOT_INT = ["n", "batches", "gen_tokens", "pad_in", "pad_out", "kv_bytes_max", "dp_cost", "viol_alone",
           "viol_seq", "over_cap", "makespan_us"]
REL = 1e-6


def gpu_run(inp, out, slo, cfg, per_batch=True):
    from paper_2409_14961_b200.scheduler import GpuScheduler
    dev = torch.device("cuda:0")
    g = GpuScheduler(len(inp), cfg, device=dev, per_batch=per_batch)
    g.run(torch.from_numpy(np.ascontiguousarray(inp).view(np.int32)).to(dev),
          torch.from_numpy(np.ascontiguousarray(out).view(np.int32)).to(dev),
          torch.from_numpy(np.ascontiguousarray(slo)).to(dev))
    r = g.results()
    r["diag"] = g.diagnostics()
    return r


def assert_parity(inp, out, slo, cfg, stats=True, nthreads=8):
    r = gpu_run(inp, out, slo, cfg, per_batch=stats)
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp, out, slo, cfg, nthreads=nthreads)
    assert np.array_equal(r["order"], o_order), "order"
    assert r["m"] == o_m, ("num_batches", r["m"], o_m)
    assert np.array_equal(r["offsets"], o_offs), "batch_offsets"
    if cfg.mode == W.MODE_SEG_DP:
        assert r["diag"]["dp_cost"] == o_cost, ("dp_cost", r["diag"]["dp_cost"], o_cost)
    if stats:
        pb, tot = oracle.stats(inp, out, slo, cfg, o_order, o_offs)
        for f in INT_FIELDS:
            assert np.array_equal(r["per_batch"][f], pb[f]), f
        for f in TOT_INT:
            assert r["totals"][f] == tot[f], (f, r["totals"][f], tot[f])
        for f in ("mean_latency_s", "throughput_tok_s"):
            assert r["totals"][f] == pytest.approx(tot[f], rel=REL, abs=0), f
        if cfg.mode == W.MODE_SEG_DP:
            assert r["totals"]["dp_cost"] == o_cost
        # the exact latency numerator the totals carry (sum over batches of b * completion_us)
        want = int((pb["size"].astype(object) * pb["completion_us"].astype(object)).sum()) if len(pb) else 0
        assert r["totals"]["latency_sum_us"] == want and r["totals"]["overflow"] == 0
    return r


# ------------------------------------------------------------------ tiny / brute-force size
@pytest.mark.parametrize("pattern", ["rand", "ties", "bucket", "identical", "descending", "classes"])
def test_small_random(pattern):
    for seed in range(40):
        n = 1 + seed % 12
        inp, out, slo, cfg = W.random_small(seed * 13 + 5, n, pattern)
        assert_parity(inp, out, slo, cfg)


@pytest.mark.parametrize("seed", range(0, 60, 3))
def test_c1(seed):
    for lam in (0, 10**6):
        assert_parity(*W.c1(seed, lam))


# ------------------------------------------------------------------ configs c2 / c3
@pytest.mark.parametrize("lam,split", [(0, 0), (10**9, 0), (10**9, 1), (0, 1)])
def test_c2(lam, split):
    assert_parity(*W.c2(7, lam=lam, split=split))


@pytest.mark.parametrize("lam", [0, 10**9])
def test_c3(lam):
    r = assert_parity(*W.c3(3, lam=lam), nthreads=1)
    assert r["diag"]["tiles"] > 1


def test_c3_windows_ragged():
    inp, out, slo, cfg = W.c3(4, n=333_333)
    assert_parity(inp, out, slo, cfg.replace(window=50_000))


# ------------------------------------------------------------------ tiling / fix-up / cascade
@pytest.mark.parametrize("W_,tile", [(64, 128), (64, 192), (256, 512), (16, 32)])
def test_forced_small_tiles(W_, tile):
    """Tiles of 2-3 W rarely converge, so the fix-up cascade and the traceback re-walks run."""
    inp, out, slo, cfg = W.c2(11, n=20_000)
    cfg = cfg.replace(max_batch=W_, dp_tile=tile)
    r = assert_parity(inp, out, slo, cfg)
    d = r["diag"]
    assert d["tiles"] >= 20_000 // (2 * tile)
    assert d["fixup_positions"] > 0


def test_identical_keys_tiles():
    # c5-i: identical keys never converge off-phase; tiles are W-aligned so they do
    n = 50_000
    inp = np.full(n, 128, np.uint32); out = np.full(n, 256, np.uint32); slo = np.full(n, 30.0, np.float32)
    cfg = W.SchedConfig(max_batch=256, kv_cap_bytes=W.C5_KV_CAP_BYTES, lambda_us=10**9, dp_tile=1024)
    assert_parity(inp, out, slo, cfg)
    assert_parity(inp, out, slo, cfg.replace(kv_cap_bytes=0, dp_tile=768))


@pytest.mark.parametrize("case", ["cap42", "windows", "viol_mid", "all_viol", "w64_nocap", "tiny_tiles",
                                  "split", "lam0", "w512"])
def test_uniform_runs_periodic_fill(case):
    """Runs of identical queries between other queries (c5-(i) embedded at an arbitrary DP phase):
    the periodic fill of uniform stretches (DESIGN.md SEG-DP step 8) must reproduce the oracle
    exactly -- local runs, parallel fix-ups (args by direct scan) and cascade re-runs (trusted
    source args), the list re-built after a stretch, every cost regime of the run's batches."""
    kw = {}
    runs = ((3_000, 128, 257), (20_000, 64, 513), (1_500, 7, 33))
    cfg_kw = {}
    if case == "windows":
        kw["window"] = 50_000
    if case == "viol_mid":
        kw["slo_s"] = 0.8              # est(b) > 0.8 s from b = 25 on: batches of 24 avoid the penalty
    if case == "all_viol":
        kw["slo_s"] = 0.3              # every batch of the 513-output run violates
    if case == "w64_nocap":
        kw["W"] = 64
        kw["cap_tokens"] = 0
    if case == "tiny_tiles":
        cfg_kw["dp_tile"] = 512        # 2 W: fix-up look-back at its lower limit, many cascade re-runs
    if case == "split":
        cfg_kw["split_on_slo_change"] = 1
    if case == "lam0":
        kw["lam"] = 0
    if case == "w512":
        kw["W"] = 512
        kw["cap_tokens"] = 1_000_000
        runs = ((9_000, 128, 257), (4_000, 3, 5))
    inp, out, slo, cfg = W.uniform_runs(31, n=150_000, runs=runs, **kw)
    if case == "w64_nocap":
        cfg = cfg.replace(kv_cap_bytes=0)
    r = assert_parity(inp, out, slo, cfg.replace(**cfg_kw))
    assert r["diag"]["dp_filled_positions"] > 0


@pytest.mark.parametrize("case", ["many_tiles", "windows", "tile_1000", "w64", "no_cap"])
def test_uniform_long_runs_deferred(case):
    """Uniform stretches spanning many DP tiles: the cascade defers every tile past the first periodic
    one to k_dp_fill (reference frame, parallel fill), materialises the tail where a re-run leaves
    the stretch or the window ends inside it; the traceback's B-walks never merge there, so the exit
    maps + parallel re-marking carry the true path through (DESIGN.md SEG-DP step 8, a7)."""
    kw = {}
    cfg_kw = {"dp_tile": 4096}
    runs = ((70_000, 128, 257), (45_000, 64, 513), (9_000, 7, 33))
    if case == "windows":
        kw["window"] = 90_000          # window ends cut the runs (stretch tails at window ends)
    if case == "tile_1000":
        cfg_kw["dp_tile"] = 1000       # tile length not a multiple of the period
    if case == "w64":
        kw["W"] = 64
    if case == "no_cap":
        kw["cap_tokens"] = 0           # period W (batches of W) instead of the cap's 42
    inp, out, slo, cfg = W.uniform_runs(33, n=260_000, runs=runs, **kw)
    if case == "no_cap":
        cfg = cfg.replace(kv_cap_bytes=0)
    r = assert_parity(inp, out, slo, cfg.replace(**cfg_kw))
    d = r["diag"]
    assert d["dp_filled_positions"] > 100_000, d
    assert d["cascade_reruns"] < d["tiles"] // 4, d


@pytest.mark.parametrize("W_", [16, 64, 256])
def test_zero_cost_full_candidate_list(W_):
    """Every service-time term and the penalty zero: every batch costs 0, no candidate dominates
    another, so after each block's prune all W + 1 candidates (b = 0 .. W) are alive and the block
    appends 32 more -- the candidate list at its largest (slot capacity W + 33).  The tie rule
    (smallest minimising i) then picks batches of W from the window start."""
    inp, out, slo, cfg = W.c3(8, n=30_000)
    cfg = cfg.replace(max_batch=W_, kv_cap_bytes=0, lambda_us=0, t_batch_us=0, t_iter_us=0, t_tok_us=0,
                      t_prefill_us=0, window=10_000)
    assert_parity(inp, out, slo, cfg)


def test_uniform_runs_generic_path_exact():
    """The generic 64-bit path has no periodic fill (slow but exact): same schedule."""
    inp, out, slo, cfg = W.uniform_runs(32, n=40_000, runs=((6_000, 128, 257),))
    assert_parity(inp, out, slo, cfg.replace(flags=1))


def test_all_violating_and_over_cap():
    inp, out, slo, cfg = W.c5(2, n=40_000, window=10_000)
    r = assert_parity(inp, out, slo, cfg)
    assert r["totals"]["over_cap"] > 0 and r["totals"]["viol_alone"] > 0


# ------------------------------------------------------------------ other modes
def test_modes_fifo_sortonly():
    inp, out, slo, cfg = W.c2(5, n=5000)
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_FIFO, window=1234))
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_SORT_ONLY))


@pytest.mark.parametrize("w1,w2,thr,split", [(1.0, 0.0, 300.0, 0), (0.0, 1.0, 500.0, 0),
                                             (1.0, 0.01, 800.0, 1), (0.5, 0.5, 60.0, 0)])
def test_mode_slo_odbs(w1, w2, thr, split):
    inp, out, slo, cfg = W.c2(9, n=8000, split=split)
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_SLO_ODBS, w1=w1, w2=w2, threshold=thr, window=3000))


@pytest.mark.parametrize("w1,w2,thr,eps", [(0.1, 0.0, 90.0, 1e-9), (0.3, 0.0, 270.0, 1e-9), (1.0, 0.0, 4096.0, 1e-9),
                                           (0.0, 1e-9, 5.0, 0.7), (1.0, 0.02, float("inf"), 1e-9)])
def test_mode_slo_odbs_cap_edges(w1, w2, thr, eps):
    """Line-20 cap = floor(threshold / max(CM, eps)) near integer quotients (w1 = 0.1, 0.3 with
    threshold = 900 w1: RN(w1 len) makes threshold/den land within an ulp of 900/len whenever len
    divides 900), exact integer quotients, den = eps, infinite threshold (threshold, eps > 0 by contract):
    the kernel's division-free flush test must decide exactly like the division."""
    inp, out, slo, cfg = W.c2(21, n=6000)
    out = out.copy()
    out[::7] = np.array([100, 150, 180, 225, 300, 450, 900, 60, 75, 90], np.uint32)[np.arange(len(out[::7])) % 10]
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_SLO_ODBS, w1=w1, w2=w2, threshold=thr, eps=eps,
                                             window=2500))


@pytest.mark.parametrize("l1,l2,additive,split", [(1.0, 1.0, 1, 0), (0.5, 2.0, 0, 1), (1.3, 0.7, 1, 1), (2.0, 1.0, 0, 0)])
def test_mode_slo_odbs_eq_variants(l1, l2, additive, split):
    """Alg. 1 with the Eq. 1/2 scale factors l1, l2 != 1 (the kernel skips the multiplications
    only when both are 1), the additive Eq. 2 reading and the SLO-change split."""
    inp, out, slo, cfg = W.c2(23, n=7000, split=split)
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.02, threshold=900.0, l1=l1, l2=l2,
                                             eq2_additive=additive, window=3000))


@pytest.mark.parametrize("W_", [1024, 2048, 4096])
def test_mode_slo_odbs_large_max_batch(W_):
    """Alg. 1 with W at and above the chain sub-tile (sub-tile = next power of two >= W: the
    shared-memory staging of the marking kernel no longer fits and it walks global memory)."""
    inp, out, slo, cfg = W.c2(24, n=12_000)
    assert_parity(inp, out, slo, cfg.replace(mode=W.MODE_SLO_ODBS, w1=0.001, w2=0.0001, threshold=1e5,
                                             max_batch=W_, window=7000))


# ------------------------------------------------------------------ edges and errors
def test_edges():
    for n in (1, 2, 3, 31, 32, 33):
        inp, out, slo, cfg = W.c2(n, n=n)
        assert_parity(inp, out, slo, cfg)
    inp, out, slo, cfg = W.c2(1, n=700)
    assert_parity(inp, out, slo, cfg.replace(max_batch=1))
    assert_parity(inp, out, slo, cfg.replace(max_batch=4096))


def test_empty():
    from paper_2409_14961_b200.scheduler import GpuScheduler
    g = GpuScheduler(0, W.SchedConfig(), device="cuda:0")
    z = torch.zeros(0, dtype=torch.int32, device="cuda:0")
    g.run(z, z, torch.zeros(0, dtype=torch.float32, device="cuda:0"))
    r = g.results()
    assert r["m"] == 0 and list(r["offsets"]) == [0]
    assert r["totals"]["n"] == 0 and r["totals"]["batches"] == 0


def test_contract_and_config_errors():
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    inp, out, slo, cfg = W.c2(0, n=100)
    g = GpuScheduler(100, cfg, device="cuda:0")
    for bad in ("in", "out", "slo_nan", "slo_neg", "slo_zero_us"):
        i2, o2, s2 = inp.copy(), out.copy(), slo.copy()
        if bad == "in": i2[5] = 0
        if bad == "out": o2[99] = 0
        if bad == "slo_nan": s2[0] = np.nan
        if bad == "slo_neg": s2[3] = -1.0
        if bad == "slo_zero_us": s2[7] = 4e-7
        with pytest.raises(U.UellmError) as e:
            g.load(torch.from_numpy(i2.view(np.int32)).cuda(), torch.from_numpy(o2.view(np.int32)).cuda(),
                   torch.from_numpy(s2).cuda())
        assert e.value.status == U.ERR_CONTRACT
    # cost bound overflow
    g2 = GpuScheduler(100, cfg.replace(lambda_us=2**62), device="cuda:0")
    with pytest.raises(U.UellmError) as e:
        g2.load(torch.from_numpy(inp.view(np.int32)).cuda(), torch.from_numpy(out.view(np.int32)).cuda(),
                torch.from_numpy(slo).cuda())
    assert e.value.status == U.ERR_OVERFLOW


def test_host_buffers_end_to_end():
    """The C-ABI with HOST buffers (staging inside the library) equals the device path."""
    from paper_2409_14961_b200.scheduler import schedule_host
    inp, out, slo, cfg = W.c3(8, n=200_000)
    cfg = cfg.replace(window=64_000)
    order, offs, m, tot = schedule_host(inp, out, slo, cfg, device="cuda:0")
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp, out, slo, cfg, nthreads=8)
    assert np.array_equal(order, o_order) and np.array_equal(offs, o_offs) and m == o_m
    assert tot["dp_cost"] == o_cost


def test_repeat_schedule_same_profile():
    """schedule/stats can be re-run on one loaded profile (keys are kept in the workspace)."""
    from paper_2409_14961_b200.scheduler import GpuScheduler
    inp, out, slo, cfg = W.c2(2, n=6000)
    g = GpuScheduler(6000, cfg, device="cuda:0")
    g.run(torch.from_numpy(inp.view(np.int32)).cuda(), torch.from_numpy(out.view(np.int32)).cuda(),
          torch.from_numpy(slo).cuda())
    a = g.results()
    g.schedule(); g.stats()
    b = g.results()
    assert np.array_equal(a["offsets"], b["offsets"]) and a["totals"] == b["totals"]


# ------------------------------------------------------------------ full sizes (sampled)
def _window_sample_parity(inp, out, slo, cfg, r, windows):
    """Windows are independent (O1): the oracle recomputes sampled windows one by one and
    they must match the GPU's full-size run bit for bit."""
    import concurrent.futures as cf
    import os
    wl = cfg.window
    offs = r["offsets"].astype(np.int64)
    c = cfg.replace(window=0)

    def orc(w):                  # (ctypes releases the GIL: windows run on all host cores)
        a, z = w * wl, min(len(inp), (w + 1) * wl)
        o = oracle.schedule(inp[a:z], out[a:z], slo[a:z], c)
        return o, oracle.stats(inp[a:z], out[a:z], slo[a:z], c, o[0], o[1])
    with cf.ThreadPoolExecutor(max_workers=min(len(windows), os.cpu_count() or 1)) as ex:
        res = dict(zip(windows, ex.map(orc, windows)))
    for w in windows:
        a, z = w * wl, min(len(inp), (w + 1) * wl)
        (o_order, o_offs, o_m, o_cost), (o_pb, o_tot) = res[w]
        assert np.array_equal(r["order"][a:z], o_order + a), w
        sel = offs[(offs >= a) & (offs <= z)]
        assert np.array_equal(sel, o_offs.astype(np.int64) + a), w
        pb = r["per_batch"]
        mine = pb[(pb["start"] >= a) & (pb["start"] < z)]
        # every per-batch record element by element; the window-local oracle run differs only in
        # the position base (start + a) and the window index (+ w); completion_us restarts at
        # every window in both (R17)
        assert len(mine) == len(o_pb), w
        for f in INT_FIELDS:
            want = o_pb[f].astype(np.int64)
            if f == "start":
                want = want + a
            if f == "window":
                want = want + w
            assert np.array_equal(mine[f].astype(np.int64), want), (w, f)
        assert int(mine["est_us"].sum()) == o_tot["makespan_us"]
        assert int((mine["est_us"] + cfg.lambda_us * mine["viol_alone"].astype(np.uint64)).sum()) == o_cost


def _global_properties(n, cfg, r):
    offs = r["offsets"].astype(np.int64)
    assert offs[0] == 0 and offs[-1] == n and np.all(np.diff(offs) > 0)
    assert np.all(np.diff(offs) <= cfg.max_batch)
    wl = cfg.window or n
    assert set(range(0, n, wl)) <= set(offs.tolist())          # windows start batches
    pb = r["per_batch"]
    assert int(pb["size"].sum()) == n
    if cfg.kv_cap_bytes:
        assert np.all((pb["kv_bytes"] <= cfg.kv_cap_bytes) | (pb["size"] == 1))
    assert r["totals"]["dp_cost"] == r["diag"]["dp_cost"]      # stats recompute == DP optimum
    o = r["order"]
    assert np.array_equal(np.sort(o), np.arange(n, dtype=np.uint32))


@pytest.mark.slow
def test_c4_full_size_sampled():
    """BJ configs[3] at its full size (10^8 queries, 10^6-query windows) in bench.py's launch
    configuration; three windows re-derived by the oracle, global invariants on all."""
    inp, out, slo, cfg = W.c4(0)
    r = gpu_run(inp, out, slo, cfg)
    _global_properties(len(inp), cfg, r)
    _window_sample_parity(inp, out, slo, cfg, r, [0, 13, 26, 41, 57, 70, 88, 99])


@pytest.mark.slow
def test_c5_full_size_all_windows():
    """BJ configs[4] at full size (10^7 adversarial queries): every one of the 10 windows is
    oracle-identical, per-batch record by record (the identical-key windows go through the
    periodic fill)."""
    inp, out, slo, cfg = W.c5(0)
    r = gpu_run(inp, out, slo, cfg)
    _global_properties(len(inp), cfg, r)
    _window_sample_parity(inp, out, slo, cfg, r, list(range(10)))
    assert r["diag"]["dp_filled_positions"] > 0


@pytest.mark.parametrize("gen", [lambda: W.c2(3, n=20_000), lambda: W.c3(6, n=150_000)])
def test_generic_64bit_path(gen):
    """flags bit 0 forces the generic 64-bit SEG-DP kernels: identical results."""
    inp, out, slo, cfg = gen()
    assert_parity(inp, out, slo, cfg.replace(flags=1, dp_tile=4 * cfg.max_batch))
    assert_parity(inp, out, slo, cfg.replace(flags=0, dp_tile=4 * cfg.max_batch))


def test_wide_values_take_generic_path():
    """lengths >= 2^16 disable the 32-bit fast path automatically."""
    inp, out, slo, cfg = W.c2(4, n=3000)
    inp = inp.copy(); inp[::97] = 70_000
    assert_parity(inp, out, slo, cfg.replace(kv_cap_bytes=0, lambda_us=0))


@pytest.mark.parametrize("world,n,window", [(4, 400_000, 30_000), (3, 100_003, 7_000), (8, 50_000, 20_000)])
def test_sharded_ranks_equal_single_run(world, n, window):
    """T5 on one GPU: the window blocks of `world` emulated ranks, each scheduled alone and packed by
    uellm_exchange_pack, combined by uellm_exchange_combine after the (emulated) allgather, give
    exactly the single-run batch_offsets and totals -- and agree with the test-side reference of
    the record format (tests/xchg_ref.py).  (8, 50_000, 20_000): ranks with empty ranges."""
    from paper_2409_14961_b200 import distributed as D
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    from tests import xchg_ref as X
    inp, out, slo, cfg = W.c3(12, n=n)
    cfg = cfg.replace(window=window)
    full = gpu_run(inp, out, slo, cfg)
    xs = [D.Exchange(n, window, world, r, "cuda:0") for r in range(world)]
    recs = []
    for r in range(world):
        a, z = xs[r].q0, xs[r].q1
        g = GpuScheduler(z - a, cfg, device="cuda:0")
        g.run(torch.from_numpy(inp[a:z].view(np.int32)).cuda(), torch.from_numpy(out[a:z].view(np.int32)).cuda(),
              torch.from_numpy(slo[a:z]).cuda())
        xs[r].pack(g.profile, g.cfg, g.totals)
        recs.append(xs[r].record.clone())
        if z > a:
            part = g.results()
            assert np.array_equal(part["order"].astype(np.int64) + a, full["order"][a:z].astype(np.int64))
    gathered = torch.cat(recs)                          # what all_gather_into_tensor delivers
    x0 = xs[0]
    x0.gathered.copy_(gathered)
    x0.combine()
    res = x0.results()
    assert res["m"] == full["m"]
    assert np.array_equal(res["offsets"], full["offsets"])
    for f in TOT_INT:
        assert res["totals"][f] == full["totals"][f], f
    assert res["totals"]["latency_sum_us"] == full["totals"]["latency_sum_us"]
    assert res["totals"]["overflow"] == 0
    for f in ("mean_latency_s", "throughput_tok_s"):
        assert res["totals"][f] == pytest.approx(full["totals"][f], rel=1e-15), f
    # the records are in the header's format: the independent numpy reading agrees
    offs_ref, tot_ref = X.combine(gathered.view(world, -1).cpu().numpy(), x0.qb)
    assert np.array_equal(offs_ref, full["offsets"].astype(np.int64))
    for f in X.TOTAL_FIELDS:
        assert tot_ref[f] == full["totals"][f], f
    # host totals variant of the combine (synchronising)
    tot_h = U.Totals()
    import ctypes
    U.exchange_combine(x0.gathered, world, x0.n_max, x0.qb, x0.ws, x0.ws_bytes, x0.offsets, x0.num_batches,
                       ctypes.addressof(tot_h))
    assert tot_h.dp_cost == full["totals"]["dp_cost"]


def test_sort_paths_compressed_and_generic():
    """Class-valued SLOs take the rank-compressed 32-bit sort key; the paper's own protocol
    (SLO uniform in [1, 350] s) overflows the distinct-value set and takes the 64-bit key.
    Both must give the oracle's order; 1024 distinct values is the largest compressed case."""
    inp, out, slo, cfg = W.c3(21, n=120_000)
    r = assert_parity(inp, out, slo, cfg.replace(window=40_000))
    assert r["diag"]["sort_key_bits"] < 32
    slo_u = W.gen_uniform_slo(120_000, 21)
    r = assert_parity(inp, out, slo_u, cfg.replace(window=40_000))
    assert r["diag"]["sort_key_bits"] == 64
    for k, expect_compressed in ((1024, True), (1025, False)):
        rng = np.random.default_rng(k)
        vals = np.sort(rng.choice(np.arange(1, 200_000), size=k, replace=False)).astype(np.float32) * np.float32(1e-3)
        s2 = vals[rng.integers(0, k, size=60_000)]
        if k == 1024:
            s2[:k] = vals
        else:
            s2[:k] = vals
        r = assert_parity(inp[:60_000], out[:60_000], s2, cfg.replace(window=0))
        assert (r["diag"]["sort_key_bits"] < 64) == expect_compressed


@pytest.mark.parametrize("split", [0, 1])
def test_mode_slo_odbs_large(split):
    """Parallel Alg. 1 (next() per position + chunked chain walk) on several windows and chunks."""
    inp, out, slo, cfg = W.c3(15, n=300_000, split=split)
    cfg = cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.02, threshold=900.0, window=70_000, max_batch=128)
    assert_parity(inp, out, slo, cfg)


def test_mode_slo_odbs_single_window_many_tiles():
    inp, out, slo, cfg = W.c2(16, n=250_000)
    cfg = cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.05, threshold=400.0, window=0)
    assert_parity(inp, out, slo, cfg, nthreads=1)


@pytest.mark.parametrize("n,window,groups", [(2_000_000, 100_000, 0), (1_234_567, 100_000, 3),
                                             (300_000, 0, 0), (250_000, 60_000, 64)])
def test_pipelined_host_end_to_end(n, window, groups):
    """uellm_schedule_pipelined (window groups overlapped with the PCIe copies) gives the oracle's
    whole-job schedule and totals from pinned host buffers."""
    from paper_2409_14961_b200 import uellm as U
    inp, out, slo, cfg = W.c3(17, n=n)
    cfg = cfg.replace(window=window)
    c = U.make_config(cfg)
    wsb = U.pipeline_workspace_bytes(n, c, groups)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    p_in = torch.from_numpy(inp.view(np.int32)).pin_memory()
    p_out = torch.from_numpy(out.view(np.int32)).pin_memory()
    p_slo = torch.from_numpy(slo).pin_memory()
    h_order = torch.empty(n, dtype=torch.int32).pin_memory()
    h_offs = torch.empty(n + 1, dtype=torch.int32).pin_memory()
    nb = np.zeros(1, np.uint64)
    tot = U.Totals()
    import ctypes
    U.schedule_pipelined(n, p_in, p_out, p_slo, c, groups, ws, wsb, h_order, h_offs, nb, ctypes.addressof(tot))
    m = int(nb[0])
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp, out, slo, cfg, nthreads=8)
    assert m == o_m
    assert np.array_equal(h_order.numpy().view(np.uint32), o_order)
    assert np.array_equal(h_offs.numpy().view(np.uint32)[: m + 1], o_offs)
    _, o_tot = oracle.stats(inp, out, slo, cfg, o_order, o_offs)
    t = tot.as_dict()
    for f in TOT_INT:
        assert t[f] == o_tot[f], f
    assert t["dp_cost"] == o_cost
    for f in ("mean_latency_s", "throughput_tok_s"):
        assert t[f] == pytest.approx(o_tot[f], rel=1e-12), f


def test_pipelined_contract_error():
    from paper_2409_14961_b200 import uellm as U
    inp, out, slo, cfg = W.c3(18, n=200_000)
    cfg = cfg.replace(window=50_000)
    slo = slo.copy()
    slo[170_000] = 0.0                       # in the last group
    c = U.make_config(cfg)
    wsb = U.pipeline_workspace_bytes(len(inp), c, 4)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    tot = U.Totals()
    with pytest.raises(U.UellmError) as e:
        U.schedule_pipelined(len(inp), inp, out, slo, c, 4, ws, wsb, np.zeros(len(inp), np.uint32),
                             np.zeros(len(inp) + 1, np.uint32), np.zeros(1, np.uint64),
                             __import__("ctypes").addressof(tot))
    assert e.value.status == U.ERR_CONTRACT


@pytest.mark.parametrize("uniform_slo", [False, True])
def test_sort_window_groups(uniform_slo, monkeypatch):
    """The sort's window-group path (a tuning knob, UELLM_SORT_GROUP_Q) gives the same order on
    both key layouts."""
    inp, out, slo, cfg = W.c3(19, n=400_000)
    if uniform_slo:
        slo = W.gen_uniform_slo(400_000, 19)
    monkeypatch.setenv("UELLM_SORT_GROUP_Q", "90000")
    assert_parity(inp, out, slo, cfg.replace(window=30_000))


def _bench_line(root, args, world=1, port=29517):
    import json
    import os
    import subprocess
    import sys
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py")]
    else:
        cmd = [sys.executable, os.path.join(root, "bench.py")]
    r = subprocess.run(cmd + args, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


@pytest.mark.parametrize("world", [2, 3])
def test_bench_ranks_one_gpu_gloo_equal_single_rank(world):
    """bench.py's N > 1 path (one job sharded by window blocks, a9 exchange through the library,
    max-over-ranks timing) with `world` ranks sharing the one GPU over gloo: the rebuilt job's
    batch_offsets + totals hash equals the single-rank run's, and the job cost is the oracle's."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = 2_000_000
    common = ["--steps", "2", "--warmup", "1", "--queries", str(n), "--no-cpu-baseline", "--no-sim", "--no-configs"]
    one = _bench_line(root, ["--gpus", "1"] + common)
    many = _bench_line(root, ["--gpus", str(world), "--dist-backend", "gloo"] + common, world=world, port=29517 + world)
    assert many["n_gpus"] == world and many["scaling"] == "strong" and many["e2e"] is not None
    assert many["config"]["queries"] == n and many["weak_scaling"] is not None
    assert many["job_offsets_sha256"] == one["job_offsets_sha256"]
    assert many["dp_cost"] == one["dp_cost"] and many["batches"] == one["batches"]
    inp, out, slo, cfg = W.c4(seed=0, n=n)
    o = oracle.schedule(inp, out, slo, cfg, nthreads=8)
    assert one["dp_cost"] == o[3] and one["batches"] == o[2]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    """T6: compute-sanitizer finds no error in a small run of every entry point.
    Opt-in (UELLM_SANITIZE=1): the GPU pool this build is tested on closed compute-sanitizer (runs
    under it left GPUs needing a reset); the four tools ran clean in rounds 1-2."""
    import os
    import subprocess
    import sys
    if os.environ.get("UELLM_SANITIZE") != "1":
        pytest.skip("compute-sanitizer is closed on this GPU pool; set UELLM_SANITIZE=1 to run it")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = ["/usr/local/cuda/bin/compute-sanitizer", "--tool", tool, "--error-exitcode", "9",
           sys.executable, os.path.join(root, "tools", "sanitize_run.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=root)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0 and "SANITIZE_RUN_OK" in r.stdout, tail
    out = r.stdout + r.stderr
    assert "ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out, tail



# ------------------------------------------------------------------ asynchronous reload + CUDA graph
def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32 if a.dtype != np.float32 else np.float32)).cuda()


def test_profile_reload_statuses_and_parity():
    """uellm_profile_reload: device-side validation against the profile's decisions (uellm.h)."""
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    inp, out, slo, cfg = W.c3(5, n=120_000)
    cfg = cfg.replace(window=30_000)
    g = GpuScheduler(len(inp), cfg, device="cuda:0")
    g.load(_dev(inp), _dev(out), _dev(slo))
    # a permutation of the same queries: same maxima, SLO set and key bits -> OK, oracle parity
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(inp))
    p_in, p_out, p_slo = inp[perm], out[perm], slo[perm]
    g.reload(_dev(p_in), _dev(p_out), _dev(p_slo))
    g.schedule()
    g.stats()
    assert int(g.status_word().item()) == U.OK
    r = g.results()
    o_order, o_offs, o_m, o_cost = oracle.schedule(p_in, p_out, p_slo, cfg, nthreads=8)
    assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs)
    assert r["totals"]["dp_cost"] == o_cost
    # a larger input length than the profile recorded -> STALE
    b_in = p_in.copy(); b_in[7] = inp.max() + 1
    g.reload(_dev(b_in), _dev(p_out), _dev(p_slo))
    assert int(g.status_word().item()) == U.ERR_STALE
    # an invalid query -> CONTRACT
    z_in = p_in.copy(); z_in[11] = 0
    g.reload(_dev(z_in), _dev(p_out), _dev(p_slo))
    assert int(g.status_word().item()) == U.ERR_CONTRACT
    # an SLO value outside the profile's set -> STALE (the rank-compressed key was decided for the set)
    s2 = p_slo.copy(); s2[5] = 123.0
    g.reload(_dev(p_in), _dev(p_out), _dev(s2))
    assert int(g.status_word().item()) == U.ERR_STALE
    # a subset of the profile's SLO values (one class folded into another) -> OK: the fused reload
    # packs with the profile's rank table; scheduling twice reuses the kept keys / histogram
    s3 = p_slo.copy(); s3[s3 == np.unique(slo)[2]] = np.unique(slo)[5]
    g.reload(_dev(p_in), _dev(p_out), _dev(s3))
    g.schedule()
    assert int(g.status_word().item()) == U.OK
    first = g.results()
    g.schedule()
    g.stats()
    r = g.results()
    o_order, o_offs, o_m, o_cost = oracle.schedule(p_in, p_out, s3, cfg, nthreads=8)
    assert np.array_equal(first["order"], o_order) and np.array_equal(first["offsets"], o_offs)
    assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs)
    assert r["totals"]["dp_cost"] == o_cost


def test_profile_reload_generic_key_path():
    """Reload of a profile with more distinct SLO values than the compressed key takes (u64 keys,
    the unfused load kernel): a permutation is OK with oracle parity, a larger maximum STALE."""
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    n = 60_000
    inp, out, _ = W.long_tail(n, 4)
    slo = W.gen_uniform_slo(n, 4)
    cfg = W.SchedConfig(window=20_000, max_batch=128, kv_cap_bytes=W.KV_RESERVE_LLAMA2_7B_180GB, lambda_us=10**9)
    g = GpuScheduler(n, cfg, device="cuda:0")
    g.load(_dev(inp), _dev(out), _dev(slo))
    perm = np.random.default_rng(5).permutation(n)
    g.reload(_dev(inp[perm]), _dev(out[perm]), _dev(slo[perm]))
    g.schedule()
    g.stats()
    assert int(g.status_word().item()) == U.OK
    r = g.results()
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp[perm], out[perm], slo[perm], cfg, nthreads=8)
    assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs)
    assert r["totals"]["dp_cost"] == o_cost and g.diagnostics()["sort_key_bits"] == 64
    # (the distinct set overflowed the compressed key: its exact size is not tracked, and the u64 key
    # does not depend on it) -- a larger output length is STALE
    o2 = out[perm].copy(); o2[3] = out.max() + 1
    g.reload(_dev(inp[perm]), _dev(o2), _dev(slo[perm]))
    assert int(g.status_word().item()) == U.ERR_STALE


def test_cuda_graph_step_equals_eager():
    """reload -> schedule -> stats captured once in a CUDA graph and replayed on new queries gives the
    eager results (every decision lives in the profile; no host synchronisation inside the step)."""
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    inp, out, slo, cfg = W.c3(6, n=200_000)
    cfg = cfg.replace(window=50_000)
    n = len(inp)
    st = torch.cuda.Stream()
    d_in, d_out, d_slo = _dev(inp), _dev(out), _dev(slo)
    g = GpuScheduler(n, cfg, device="cuda:0")
    g.load(d_in, d_out, d_slo, st)
    torch.cuda.synchronize()
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg, stream=st, capture_error_mode="thread_local"):
        g.reload(d_in, d_out, d_slo, st)
        g.schedule(st)
        g.stats(st)
    rng = np.random.default_rng(9)
    for it in range(3):
        perm = rng.permutation(n)
        d_in.copy_(_dev(inp[perm])); d_out.copy_(_dev(out[perm])); d_slo.copy_(_dev(slo[perm]))
        cg.replay()
        torch.cuda.synchronize()
        assert int(g.status_word().item()) == U.OK
        r = g.results()
        o_order, o_offs, o_m, o_cost = oracle.schedule(inp[perm], out[perm], slo[perm], cfg, nthreads=8)
        assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs), it
        assert r["totals"]["dp_cost"] == o_cost
