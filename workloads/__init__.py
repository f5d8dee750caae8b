"""Seeded synthetic query streams and scheduler configurations (c1-c5).

This module is shared INPUT plumbing: both the CPU oracle (oracle/) and the CUDA path
(paper_2409_14961_b200/) are fed from it, so it deliberately contains none of the
method's arithmetic -- no SLO conversion, no sort, no cost model, no KV formula.  It
only draws numbers and states configuration constants.

Distributions are proposals (the paper publishes none):
  * SLO: "ranging from 1 second to 350 seconds"; class-valued variants for c2-c4.
  * input length: lognormal (Alpaca-like prompts, P:195 names Alpaca as the workload).
  * predicted output length: lognormal (c2) or Pareto long tail up to 4096 (c3-c5),
    quantised to the profiler's length buckets ("categorize the output lengths").
Recipe and readings: DESIGN.md section "Input recipe".

Queries are returned as three numpy arrays (caller SoA):
  input_len u32, pred_out_len u32, slo_s f32 (seconds).
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

# Segmentation modes (the numeric values of the C-ABI enum and of the oracle's enum).
MODE_SEG_DP = 0
MODE_SLO_ODBS = 1
MODE_FIFO = 2
MODE_SORT_ONLY = 3

# KV reserve of LLaMA-2-7B (fp16 weights 2 * 6,738,415,616 B) on one 180 GB B200:
# T of P:366 ("memory reserved for KV Cache"), in bytes.  With 4 B/elem, 32 layers,
# hidden 4096 this is 317,617 tokens of KV.
KV_RESERVE_LLAMA2_7B_180GB = 180_000_000_000 - 2 * 6_738_415_616


@dataclass
class SchedConfig:
    """Scheduler configuration; field names and meaning follow include/uellm.h."""
    mode: int = MODE_SEG_DP
    window: int = 0                 # queries per scheduling window, 0 = all
    max_batch: int = 256            # W
    split_on_slo_change: int = 0
    kv_bytes_per_elem: int = 4      # the "4" of P:60
    n_layers: int = 32              # LLaMA-2-7B
    hidden: int = 4096
    kv_cap_bytes: int = 0           # 0 = no cap
    t_batch_us: int = 1000          # service-time model (R7)
    t_iter_us: int = 2000
    t_tok_us: int = 40
    t_prefill_us: int = 10
    lambda_us: int = 0              # penalty per violating query (R8/R14)
    w1: float = 1.0                 # Alg. 1 weights / overheads / threshold
    w2: float = 1.0
    l1: float = 1.0
    l2: float = 1.0
    threshold: float = 1000.0
    eps: float = 1e-9
    eq2_additive: int = 0
    dp_tile: int = 0                # GPU SEG-DP tile length (tuning only; 0 = automatic)
    flags: int = 0                  # GPU: bit 0 forces the generic 64-bit SEG-DP kernels (testing)

    def replace(self, **kw) -> "SchedConfig":
        return dataclasses.replace(self, **kw)


def _rng(seed: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & (2**64 - 1), stream]))


def _lognormal_int(rng, median, sigma, lo, hi, n):
    x = rng.lognormal(mean=np.log(median), sigma=sigma, size=n)
    return np.clip(np.rint(x), lo, hi).astype(np.uint32)


def _bucket_up(x, width, hi):
    x = ((x.astype(np.int64) + width - 1) // width) * width
    return np.clip(x, width, hi).astype(np.uint32)


def _pareto_out(rng, n, alpha=1.2, xm=32, hi=4096, width=16):
    x = xm * (1.0 + rng.pareto(alpha, size=n))
    x = np.minimum(np.ceil(x), hi)
    return _bucket_up(x.astype(np.int64), width, hi)


SLO_CLASSES_8 = np.geomspace(1.0, 350.0, 8).astype(np.float32)
SLO_CLASSES_3 = np.array([2.0, 30.0, 350.0], dtype=np.float32)


def gen_uniform_slo(n, seed, lo=1.0, hi=350.0):
    """The paper's own protocol: per-request SLO uniform in [1 s, 350 s]."""
    rng = _rng(seed, 7)
    return rng.uniform(lo, hi, size=n).astype(np.float32)


def c1(seed: int, lam: int = 0):
    """16 queries, 1 SLO class (0.3 s), outputs 8-128, cap = 4 queries' KV (BJ configs[0])."""
    rng = _rng(seed, 1)
    n = 16
    inp = rng.integers(1, 65, size=n).astype(np.uint32)
    out = rng.integers(8, 129, size=n).astype(np.uint32)
    slo = np.full(n, 0.3, dtype=np.float32)
    # 4 queries of the largest possible length (64 + 128 tokens) at 4*32*4096 B/token
    cap = 4 * 192 * 524_288
    cfg = SchedConfig(window=0, max_batch=16, kv_cap_bytes=cap, lambda_us=lam)
    return inp, out, slo, cfg


def c2(seed: int, lam: int = 10**9, split: int = 0, n: int = 10_000):
    """10^4 queries, 3 SLO classes, Alpaca-like lengths, W = 64 (BJ configs[1])."""
    rng = _rng(seed, 2)
    inp = _lognormal_int(rng, 24, 0.6, 1, 512, n)
    out = _bucket_up(_lognormal_int(rng, 64, 0.9, 1, 1024, n), 32, 1024)
    slo = SLO_CLASSES_3[rng.integers(0, 3, size=n)]
    cfg = SchedConfig(window=0, max_batch=64, kv_cap_bytes=KV_RESERVE_LLAMA2_7B_180GB,
                      lambda_us=lam, split_on_slo_change=split)
    return inp, out, slo, cfg


def long_tail(n: int, seed: int, stream: int = 3):
    """c3/c4 query shape: 8 log-spaced SLO classes in [1, 350] s, lognormal inputs
    (median 128, sigma 1, <= 4096), Pareto(1.2) x 32 outputs (<= 4096, 16-token buckets)."""
    rng = _rng(seed, stream)
    inp = _lognormal_int(rng, 128, 1.0, 1, 4096, n)
    out = _pareto_out(rng, n)
    slo = SLO_CLASSES_8[rng.integers(0, 8, size=n)]
    return inp, out, slo


def c3(seed: int, lam: int = 10**9, split: int = 0, n: int = 1_000_000):
    """10^6 queries, 8 SLO classes, long-tail outputs <= 4096, LLaMA-2-7B KV cap (configs[2])."""
    inp, out, slo = long_tail(n, seed)
    cfg = SchedConfig(window=0, max_batch=256, kv_cap_bytes=KV_RESERVE_LLAMA2_7B_180GB,
                      lambda_us=lam, split_on_slo_change=split)
    return inp, out, slo, cfg


def c4(seed: int, lam: int = 10**9, n: int = 100_000_000, window: int = 1_000_000):
    """10^8 queries streamed in 10^6-query windows (BJ configs[3]); shape as c3."""
    inp, out, slo = long_tail(n, seed)
    cfg = SchedConfig(window=window, max_batch=256, kv_cap_bytes=KV_RESERVE_LLAMA2_7B_180GB,
                      lambda_us=lam)
    return inp, out, slo, cfg


C5_KV_CAP_BYTES = 16_384 * 524_288   # 16,384 tokens of LLaMA-2-7B KV


def c5(seed: int, n: int = 10_000_000, window: int = 1_000_000, lam: int = 10**9):
    """Adversarial mix (BJ configs[4]), four equal contiguous segments:
      (i)   identical keys: slo 30 s, input 128, output 256;
      (ii)  all-violating: slo 1 ms (< t_batch + t_iter), c3-shaped lengths;
      (iii) 1% of queries alone exceed the KV cap (in + out in (16384, 32768]);
      (iv)  anti-sorted: strictly ascending distinct SLOs with descending outputs."""
    rng = _rng(seed, 5)
    q = n // 4
    sizes = [q, q, q, n - 3 * q]
    ins, outs, slos = [], [], []
    # (i)
    ins.append(np.full(sizes[0], 128, np.uint32))
    outs.append(np.full(sizes[0], 256, np.uint32))
    slos.append(np.full(sizes[0], 30.0, np.float32))
    # (ii)
    a, b, _ = long_tail(sizes[1], seed, stream=51)
    ins.append(a); outs.append(b); slos.append(np.full(sizes[1], 1e-3, np.float32))
    # (iii)
    a, b, c = long_tail(sizes[2], seed, stream=52)
    big = rng.random(sizes[2]) < 0.01
    nb = int(big.sum())
    tot = rng.integers(16_385, 32_769, size=nb)
    bi = np.maximum(1, (tot * rng.random(nb)).astype(np.int64))
    bi = np.minimum(bi, tot - 1)
    a = a.copy(); b = b.copy()
    a[big] = bi.astype(np.uint32)
    b[big] = (tot - bi).astype(np.uint32)
    ins.append(a); outs.append(b); slos.append(c)
    # (iv)
    m = sizes[3]
    ins.append(_lognormal_int(rng, 128, 1.0, 1, 4096, m))
    outs.append(np.linspace(4096, 1, m).astype(np.uint32))
    slos.append(np.linspace(1.0, 350.0, m, dtype=np.float64).astype(np.float32))
    inp = np.concatenate(ins); out = np.concatenate(outs); slo = np.concatenate(slos)
    cfg = SchedConfig(window=window, max_batch=256, kv_cap_bytes=C5_KV_CAP_BYTES, lambda_us=lam)
    return inp, out, slo, cfg


def uniform_runs(seed: int, n: int = 200_000, runs=((3_000, 128, 257), (20_000, 64, 513)), slo_s: float = 30.0,
                 window: int = 0, W: int = 256, cap_tokens: int = 16_384, lam: int = 10**9):
    """c3-shaped background plus maximal runs of identical queries (in, out, slo) -- the shape of
    c5-(i) (identical keys) embedded between other queries, so the run starts at an arbitrary
    phase of the DP and is followed by more work.  All queries share one SLO; each run uses an
    output length no background query has (odd values; the background is a multiple of 16), so
    after the (slo, out, idx) sort every run is contiguous and preceded and followed by other
    queries.  runs: (length, input, output) triples."""
    rng = _rng(seed, 61)
    m = n - sum(r[0] for r in runs)
    inp, out, _ = long_tail(m, seed, stream=62)
    parts_in, parts_out = [inp], [out]
    for length, ri, ro in runs:
        assert ro % 2 == 1, "run outputs must be odd (unique against the 16-bucketed background)"
        parts_in.append(np.full(length, ri, np.uint32))
        parts_out.append(np.full(length, ro, np.uint32))
    inp = np.concatenate(parts_in); out = np.concatenate(parts_out)
    perm = rng.permutation(n)
    inp, out = inp[perm], out[perm]
    slo = np.full(n, slo_s, np.float32)
    cfg = SchedConfig(window=window, max_batch=W, kv_cap_bytes=cap_tokens * 524_288, lambda_us=lam)
    return inp, out, slo, cfg


# Mean inter-arrival gaps (us) for the simulator (NEXT f2): about one query's share of the
# makespan the R7 service model gives the SEG-DP schedules of these shapes (c2 ~10 ms/query,
# c3/c4 ~21.6 ms/query), i.e. a replica loaded close to saturation.
MEAN_GAP_US = {"c2": 10_000, "c3": 21_000, "c4": 21_000}


def poisson_arrivals(n: int, seed: int, mean_gap_us: float, stream: int = 11) -> np.ndarray:
    """Arrival times (u64 us, nondecreasing in arrival index): cumulative sums of rounded
    exponential gaps (a Poisson stream; the paper states none)."""
    rng = _rng(seed, stream)
    gaps = np.rint(rng.exponential(mean_gap_us, size=n)).astype(np.int64)
    return np.cumsum(gaps).astype(np.uint64)


def random_arrivals(n: int, seed: int, hi: int, stream: int = 12) -> np.ndarray:
    """Arrivals in any order (uniform in [0, hi)): exercises batches whose latest member arrives
    after the previous batch ends."""
    rng = _rng(seed, stream)
    return rng.integers(0, max(hi, 1), size=n).astype(np.uint64)


@dataclass
class PredictorConfig:
    """Profiler stand-in + monitor configuration (NEXT f4); field names follow include/uellm.h
    (uellm_predictor).  Defaults: SPEC S:216 (gamma 1.1, cap 2.0); the noisy variant's error
    rate 0.0049 mimics the paper's 99.51 % bucket precision."""
    variant: int = 2                # 0 oracle, 1 bucketed, 2 noisy, 3 constant
    bucket_width: int = 16
    constant_tokens: int = 256
    window: int = 0
    error_rate: float = 0.0049
    gamma: float = 1.1
    cap: float = 2.0
    seed: int = 0
    monitor: int = 1

    def replace(self, **kw) -> "PredictorConfig":
        return dataclasses.replace(self, **kw)


def true_output_lengths(n: int, seed: int, stream: int = 13) -> np.ndarray:
    """True (generated) output lengths for the profiler stand-ins: the long-tail shape of c3/c4
    before bucketing (Pareto(1.2) x 32, <= 4096)."""
    rng = _rng(seed, stream)
    x = 32 * (1.0 + rng.pareto(1.2, size=n))
    return np.minimum(np.ceil(x), 4096).astype(np.uint32)


@dataclass
class Topology:
    """HELR deployer input (NEXT f3): devices, links and the model to place."""
    memory_bytes: np.ndarray            # u64 [D], Memory(d)
    performance: np.ndarray             # f64 [D], Performance(d) (> 0)
    link_latency_s: np.ndarray          # f64 [D, D], Latency(E[i][j]), symmetric, zero diagonal
    num_layers: int = 32                # Layer(M)
    model_bytes: int = 2 * 6_738_415_616     # M (LLaMA-2-7B fp16 weights)
    kv_reserve_bytes: int = 0           # T (Alg. 2 line 11)
    p: float = 1.0
    a1: float = 1.0
    a2: float = 1.0

    def replace(self, **kw) -> "Topology":
        return dataclasses.replace(self, **kw)


def b200_cluster(nodes: int = 2, per_node: int = 8, seed: int = 0, model_bytes: int = 2 * 70_553_706_496,
                 num_layers: int = 80, kv_reserve_bytes: int = 120_000_000_000) -> Topology:
    """A synthetic multi-node B200 topology for HELR: per-device free memory drawn between 140 and
    180 GB (other tenants), performance 0.85-1.0 (relative), NVLink 5 / NVSwitch inside a node
    (~2 us), InfiniBand between nodes (~10 us); default model LLaMA-2-70B fp16 (80 layers) with a
    120 GB-per-device KV reserve so that several devices are needed."""
    rng = _rng(seed, 31)
    D = nodes * per_node
    mem = rng.integers(140, 181, size=D).astype(np.uint64) * np.uint64(1_000_000_000)
    perf = rng.uniform(0.85, 1.0, size=D)
    node = np.arange(D) // per_node
    lat = np.where(node[:, None] == node[None, :], 2e-6, 10e-6) * rng.uniform(0.9, 1.1, size=(D, D))
    lat = (lat + lat.T) / 2
    np.fill_diagonal(lat, 0.0)
    return Topology(mem, perf, lat, num_layers=num_layers, model_bytes=model_bytes,
                    kv_reserve_bytes=kv_reserve_bytes, p=1e-12)


def random_topology(seed: int, D: int) -> Topology:
    """Small random topologies for the brute-force pins."""
    rng = _rng(seed, 32)
    L = int(rng.integers(1, 40))
    M = int(rng.integers(1, 100)) * L
    mem = rng.integers(0, 2 * M, size=D).astype(np.uint64)
    perf = rng.uniform(0.5, 4.0, size=D)
    lat = rng.uniform(0.0, 3.0, size=(D, D))
    if rng.random() < 0.3:
        lat = np.round(lat)                  # exact ties
    lat = (lat + lat.T) / 2
    np.fill_diagonal(lat, 0.0)
    T = int(rng.integers(0, M // 2 + 1))
    a1, a2 = [(1.0, 1.0), (0.0, 1.0), (10.0, 1.0), (1.0, 0.0)][int(rng.integers(0, 4))]
    return Topology(mem, perf, lat, num_layers=L, model_bytes=M, kv_reserve_bytes=T,
                    p=float(rng.choice([1.0, 0.5, 2.0])), a1=a1, a2=a2)


def random_small(seed: int, n: int, pattern: str = "rand"):
    """Tiny brute-force-checkable instances with a random configuration.
    pattern: rand | ties | bucket | identical | descending | classes."""
    rng = _rng(seed, 9)
    if pattern == "identical":
        inp = np.full(n, int(rng.integers(1, 50)), np.uint32)
        out = np.full(n, int(rng.integers(1, 50)), np.uint32)
        slo = np.full(n, np.float32(rng.uniform(0.001, 0.5)), np.float32)
    else:
        inp = rng.integers(1, 40, size=n).astype(np.uint32)
        out = rng.integers(1, 40, size=n).astype(np.uint32)
        if pattern == "ties":
            inp = rng.integers(1, 4, size=n).astype(np.uint32) * 8
            out = rng.integers(1, 4, size=n).astype(np.uint32) * 8
        if pattern == "bucket":
            out = (rng.integers(1, 5, size=n) * 16).astype(np.uint32)
        if pattern == "descending":
            out = np.sort(out)[::-1].copy()
        slo = rng.uniform(0.0005, 0.05, size=n).astype(np.float32)
        if pattern in ("ties", "classes", "bucket"):
            cls = np.array([0.002, 0.01, 0.03], dtype=np.float32)
            slo = cls[rng.integers(0, 3, size=n)]
        if pattern == "descending":
            slo = np.sort(slo)
    cap = int(rng.choice([0, 300, 1200, 5000, 30000]))
    cfg = SchedConfig(
        window=0,
        max_batch=int(rng.integers(1, n + 2)),
        split_on_slo_change=int(rng.integers(0, 2)),
        kv_bytes_per_elem=int(rng.choice([1, 2, 4])),
        n_layers=int(rng.integers(1, 4)),
        hidden=int(rng.integers(1, 4)),
        t_batch_us=int(rng.integers(0, 3000)),
        t_iter_us=int(rng.integers(0, 300)),
        t_tok_us=int(rng.integers(0, 50)),
        t_prefill_us=int(rng.integers(0, 20)),
        lambda_us=int(rng.choice([0, 1, 1000, 10**6, 10**9])),
    )
    cfg.kv_cap_bytes = cap
    if cfg.t_batch_us == 0 and cfg.t_iter_us == 0 and rng.random() < 0.5:
        cfg.t_batch_us = 1
    return inp, out, slo, cfg


def random_medium(seed: int):
    """Randomised medium-size instances for the GPU parity fuzz test: every SEG-DP kernel variant
    (lambda 0 / < 2^32 / >= 2^32, SLO split, many SLO runs), both sort key layouts (class-valued
    SLOs vs more than 1024 distinct values), windows of any length (16-byte aligned or not), forced
    DP tile lengths, the generic 64-bit path, KV caps that bind or not, zero service-time terms,
    uniform stretches.  Returns (inp, out, slo, cfg)."""
    rng = _rng(seed, 71)
    n = int(rng.choice([1, 2, 31, 33, 1000, 4097, 20_000, 60_000]))
    shape = str(rng.choice(["longtail", "alpaca", "runs", "identical", "distinct", "tiny"]))
    if shape == "longtail":
        inp, out, slo = long_tail(n, seed, stream=72)
    elif shape == "alpaca":
        inp = _lognormal_int(rng, 24, 0.6, 1, 512, n)
        out = _bucket_up(_lognormal_int(rng, 64, 0.9, 1, 1024, n), 32, 1024)
        slo = SLO_CLASSES_3[rng.integers(0, 3, size=n)]
    elif shape == "runs":
        inp, out, slo = long_tail(n, seed, stream=73)
        k = int(rng.integers(1, 4))
        for _ in range(k):                       # a few long stretches of one identical query
            a = int(rng.integers(0, max(1, n)))
            z = min(n, a + int(rng.integers(1, max(2, n // 2))))
            inp[a:z] = int(rng.integers(1, 300)); out[a:z] = 2 * int(rng.integers(1, 200)) + 1
            slo[a:z] = slo[a]
    elif shape == "identical":
        inp = np.full(n, int(rng.integers(1, 500)), np.uint32)
        out = np.full(n, int(rng.integers(1, 2000)), np.uint32)
        slo = np.full(n, np.float32(rng.uniform(0.5, 100.0)), np.float32)
    elif shape == "distinct":                   # > 1024 distinct SLOs: the u64 key path, many runs
        inp = _lognormal_int(rng, 128, 1.0, 1, 4096, n)
        out = rng.integers(1, 4097, size=n).astype(np.uint32)
        slo = rng.uniform(0.5, 350.0, size=n).astype(np.float32)
    else:
        inp = rng.integers(1, 40, size=n).astype(np.uint32)
        out = rng.integers(1, 40, size=n).astype(np.uint32)
        slo = rng.uniform(0.001, 0.05, size=n).astype(np.float32)
    W = int(rng.choice([1, 2, 8, 16, 64, 256, 512]))
    lam = int(rng.choice([0, 1000, 10**9, 10**10]))
    window = int(rng.choice([0, 0, 1000, 4097, 25_000, 30_000]))
    cap_tok = int(rng.choice([0, 2000, 16_384, 317_617]))
    t = [int(rng.choice(v)) for v in ([0, 1000, 1000], [0, 2000, 2000], [0, 40, 40], [0, 10, 10])]
    if t[0] == 0 and t[1] == 0 and rng.random() < 0.5:
        t[0] = 1000
    tile = 0
    if rng.random() < 0.3:
        tile = W * int(rng.choice([2, 3, 4, 8, 16]))
    cfg = SchedConfig(window=window, max_batch=W, split_on_slo_change=int(rng.integers(0, 2)),
                      kv_cap_bytes=cap_tok * 524_288, t_batch_us=t[0], t_iter_us=t[1], t_tok_us=t[2],
                      t_prefill_us=t[3], lambda_us=lam, dp_tile=tile,
                      flags=1 if rng.random() < 0.1 else 0)
    u = rng.random()
    if u < 0.15:                                # the paper's Alg. 1 (random weights / threshold)
        cfg = cfg.replace(mode=MODE_SLO_ODBS, w1=float(rng.choice([0.0, 0.3, 1.0])),
                          w2=float(rng.choice([0.02, 0.5, 1.0])), threshold=float(rng.choice([50.0, 900.0, 5000.0])),
                          l1=float(rng.choice([1.0, 2.0])), l2=float(rng.choice([1.0, 0.5])),
                          eq2_additive=int(rng.integers(0, 2)))
        if cfg.w1 + cfg.w2 == 0.0:
            cfg = cfg.replace(w2=1.0)
    elif u < 0.2:
        cfg = cfg.replace(mode=MODE_FIFO)
    elif u < 0.25:
        cfg = cfg.replace(mode=MODE_SORT_ONLY)
    return inp, out, slo, cfg
