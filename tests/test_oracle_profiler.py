"""Pins of the oracle's profiler stand-ins and misprediction monitor (oracle O9-O11, NEXT f4)
against SPEC's worked examples, its invariants (including the
statistical accuracy test of the noisy predictor) and an independent Python re-implementation of
the windowed closed loop (R20) on small streams (-m "not gpu")."""
import math

import numpy as np
import pytest

import oracle
import workloads as W

P = W.PredictorConfig


def test_spec_s205_oracle_identity():
    assert oracle.predict([37], P(variant=0, monitor=0))[0] == 37          # S:205 [TRIVIAL]


def test_spec_s206_bucket_ceiling():
    assert oracle.predict([37], P(variant=1, bucket_width=50))[0] == 50    # S:206 [DERIVED]
    assert list(oracle.predict([1, 50, 51, 100, 101], P(variant=1, bucket_width=50))) == [50, 50, 100, 100, 150]


def test_spec_s207_zero_noise_is_bucketed():
    t = W.true_output_lengths(20_000, 3)
    a = oracle.predict(t, P(variant=2, error_rate=0.0, bucket_width=16, seed=9))
    b = oracle.predict(t, P(variant=1, bucket_width=16))
    assert np.array_equal(a, b)                                            # S:207 [TRIVIAL]


def test_constant_and_inflation_round_up():
    # S:205 "then multiplied by monitor.inflation_factor and rounded up"
    assert oracle.predict([999], P(variant=3, constant_tokens=7))[0] == 7
    assert oracle.predict([37], P(variant=1, bucket_width=50), factor=1.1)[0] == math.ceil(50 * 1.1) == 56
    assert oracle.predict([37], P(variant=1, bucket_width=50), factor=2.0)[0] == 100
    # R20: saturates at 2^32 - 1
    assert oracle.predict([4_000_000_000], P(variant=0), factor=2.0)[0] == 2**32 - 1


def test_spec_s216_s218_monitor():
    assert oracle.monitor_observe([50], [40], 1.1, 2.0) == (0, 1.0)        # S:216 over-prediction is safe
    c, f = oracle.monitor_observe([50], [60], 1.1, 2.0)
    assert c == 1 and f == 1.1
    c, f = oracle.monitor_observe([50] * 20, [60] * 20, 1.1, 2.0)          # S:218 saturates at cap
    assert c == 20 and f == 2.0
    # before saturation the factor is the iterated product
    c, f = oracle.monitor_observe([1] * 5, [2] * 5, 1.1, 2.0)
    assert f == 1.0 * 1.1 * 1.1 * 1.1 * 1.1 * 1.1 and f < 2.0


def test_s224_oracle_without_monitor_is_exact():
    t = W.true_output_lengths(10_000, 4)
    pred, factors, corr = oracle.profile_stream(t, P(variant=0, monitor=0, window=1000))
    assert np.array_equal(pred, t) and corr == 0 and np.all(factors == 1.0)


def test_s225_bucketed_never_underpredicts():
    t = W.true_output_lengths(50_000, 5)
    for w in (1, 16, 50, 128):
        pred, factors, corr = oracle.profile_stream(t, P(variant=1, bucket_width=w, window=5000))
        assert np.all(pred >= t) and corr == 0
        assert np.array_equal((pred + w - 1) // w, (t + w - 1) // w)      # bucket accuracy 100 %
        assert np.all(pred % w == 0)


@pytest.mark.parametrize("e", [0.0049, 0.2, 0.5, 1.0])
def test_s226_noisy_accuracy_converges(e):
    # accuracy (predicted bucket == true bucket) -> 1 - e within 3 standard errors; the two
    # displacement directions are equally likely (lengths above the first bucket only, where both
    # directions are possible, R20)
    n = 400_000
    rng = np.random.default_rng(1)
    t = rng.integers(17, 4096, size=n).astype(np.uint32)
    pred = oracle.predict(t, P(variant=2, error_rate=e, bucket_width=16, seed=11))
    kb = (t.astype(np.int64) + 15) // 16
    kp = pred.astype(np.int64) // 16
    acc = np.mean(kb == kp)
    se = math.sqrt(max(e * (1 - e), 1e-12) / n)
    assert abs(acc - (1 - e)) <= 3 * se + 1e-12
    assert set(np.unique(kp - kb)) <= {-1, 0, 1}
    up, down = np.sum(kp - kb == 1), np.sum(kp - kb == -1)
    if e > 0:
        assert abs(up - down) <= 3 * math.sqrt(up + down)
    # reproducible and seed-dependent
    assert np.array_equal(pred, oracle.predict(t, P(variant=2, error_rate=e, bucket_width=16, seed=11)))
    if 0 < e < 1:
        assert not np.array_equal(pred, oracle.predict(t, P(variant=2, error_rate=e, bucket_width=16, seed=12)))


def _py_mix64(seed, index):
    m = (1 << 64) - 1
    z = (seed ^ (index * 0x9E3779B97F4A7C15)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _py_stream(t, pc, f0=1.0):
    """Independent Python reading of S:200-218 + R20 (window epochs)."""
    n = len(t)
    wl = pc.window or n
    pred, factors, corr, f = [], [], 0, f0
    for a in range(0, n, wl):
        factors.append(f)
        chunk = []
        for k in range(a, min(n, a + wl)):
            x = int(t[k])
            if pc.variant == 0:
                base = x
            elif pc.variant == 3:
                base = pc.constant_tokens
            else:
                b = max(1, -(-x // pc.bucket_width))
                if pc.variant == 2:
                    z = _py_mix64(pc.seed, k)
                    if (z >> 11) * 2.0 ** -53 < pc.error_rate:
                        b = b + 1 if z & 1 else max(1, b - 1)
                base = b * pc.bucket_width
            chunk.append(min(math.ceil(base * f), 2**32 - 1))
        pred += chunk
        if pc.monitor:
            for p_, x in zip(chunk, t[a:a + wl]):
                if int(x) > p_:
                    corr += 1
                    f = min(f * pc.gamma, pc.cap)
    factors.append(f)
    return pred, factors, corr


@pytest.mark.parametrize("pc", [P(variant=2, error_rate=0.3, bucket_width=32, window=700, seed=5),
                                P(variant=3, constant_tokens=40, window=500, gamma=1.05, cap=3.0),
                                P(variant=2, error_rate=1.0, bucket_width=8, window=0, seed=2),
                                P(variant=1, bucket_width=10, window=333)])
def test_stream_vs_python(pc):
    t = W.true_output_lengths(4000, 8)
    pred, factors, corr = oracle.profile_stream(t, pc)
    p2, f2, c2 = _py_stream(t, pc)
    assert list(pred) == p2 and list(factors) == f2 and corr == c2
