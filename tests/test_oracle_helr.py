"""Pins of the oracle's HELR deployer (O12, NEXT f3) against things other than itself (-m "not
gpu"): exhaustive enumeration of every feasible subset x every visit order ("brute-force
oracle"), SPEC's worked examples and invariants."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def brute_helr(t: W.Topology):
    """All ordered chains over all subsets, evaluated straight from the definitions (Python ints
    for the layer split; the chain latency summed in visit order)."""
    D = len(t.memory_bytes)
    L, M, T = t.num_layers, t.model_bytes, t.kv_reserve_bytes
    m = M / L
    cap = [0 if int(x) <= T else min(L, (int(x) - T) * L // M) for x in t.memory_bytes]
    best = None
    for k in range(1, D + 1):
        for S in itertools.combinations(range(D), k):
            if sum(cap[d] for d in S) < L:
                continue
            for perm in itertools.permutations(S):
                used, lat = 0, None
                for idx, d in enumerate(perm):
                    x = min(max(0, L - used), cap[d])
                    used += cap[d]
                    c = ((t.p * x) * m) / float(t.performance[d])
                    lat = c if idx == 0 else (lat + float(t.link_latency_s[perm[idx - 1]][d])) + c
                obj = t.a1 * lat + t.a2 * (k / D)
                key = (obj, lat)
                if best is None or key < best[0]:
                    best = (key, perm)
    return best


def chain_latency(t, devices):
    L, M, T = t.num_layers, t.model_bytes, t.kv_reserve_bytes
    cap = [0 if int(x) <= T else min(L, (int(x) - T) * L // M) for x in t.memory_bytes]
    used, lat = 0, None
    for idx, d in enumerate(devices):
        x = min(max(0, L - used), cap[d])
        used += cap[d]
        c = ((t.p * x) * (M / L)) / float(t.performance[d])
        lat = c if idx == 0 else (lat + float(t.link_latency_s[devices[idx - 1]][d])) + c
    return lat


@pytest.mark.parametrize("seed", range(120))
def test_helr_vs_exhaustive_chains(seed):
    D = 1 + seed % 6
    t = W.random_topology(seed, D)
    r = oracle.helr(t)
    b = brute_helr(t)
    if b is None:
        assert not r["feasible"]
        return
    assert r["feasible"]
    assert (r["objective"], r["latency_s"]) == b[0]            # exact: same sums in the same order
    assert chain_latency(t, r["devices"]) == r["latency_s"]   # the decoded chain realises it
    # the map covers [0, L) contiguously in visit order within each device's capacity
    assert sum(r["layer_count"]) == t.num_layers
    assert r["layer_begin"][0] == 0
    for k in range(1, len(r["devices"])):
        assert r["layer_begin"][k] == min(t.num_layers, r["layer_begin"][k - 1] + r["layer_count"][k - 1]) \
            or r["layer_count"][k] == 0
    assert r["mask"] == sum(1 << d for d in r["devices"])


def one_device(mem, perf=1.0, L=32, M=32, T=0, p=1.0):
    return W.Topology(np.array([mem], np.uint64), np.array([perf]), np.zeros((1, 1)), num_layers=L,
                      model_bytes=M, kv_reserve_bytes=T, p=p)


def test_spec_s346_compute_cost():
    # p = 1, layers = 10, m = 2 bytes, performance = 4 -> 5.0
    r = oracle.helr(one_device(mem=10**6, perf=4.0, L=10, M=20))
    assert r["latency_s"] == 5.0 and r["devices"] == [0] and r["layer_count"] == [10]


def test_spec_s354_max_layers():
    # memory 24 GB, kv reserve 4 GB, m = 1 GB, 32 layers -> 20 layers fit: a lone device
    # cannot hold the model; two such devices split 20 + 12
    G = 10**9
    t = W.Topology(np.array([24 * G, 24 * G], np.uint64), np.array([1.0, 1.0]), np.array([[0, 1e-3], [1e-3, 0]]),
                   num_layers=32, model_bytes=32 * G, kv_reserve_bytes=4 * G, p=1e-9)
    r = oracle.helr(t)
    assert r["layer_count"] == [20, 12] and sorted(r["devices"]) == [0, 1]
    assert not oracle.helr(one_device(mem=24 * G, L=32, M=32 * G, T=4 * G))["feasible"]
    assert not oracle.helr(one_device(mem=4 * G, L=32, M=32 * G, T=4 * G))["feasible"]   # S:355 no headroom


def test_spec_s372_single_device():
    r = oracle.helr(one_device(mem=100, perf=2.0, L=32, M=64, p=1.0))
    assert r["devices"] == [0] and r["layer_begin"] == [0] and r["layer_count"] == [32]
    assert r["latency_s"] == 1.0 * 32 * 2.0 / 2.0


def test_spec_s373_two_identical_devices_one_wins():
    t = W.Topology(np.array([100, 100], np.uint64), np.array([1.0, 1.0]), np.array([[0, 0.5], [0.5, 0]]),
                   num_layers=8, model_bytes=8, p=1.0, a1=1.0, a2=0.0)
    r = oracle.helr(t)
    assert len(r["devices"]) == 1 and r["latency_s"] == 8.0


@pytest.mark.parametrize("seed", range(30))
def test_he_minimal_subset_and_monotone(seed):
    t = W.random_topology(seed, 5)
    he = oracle.helr(t.replace(a1=0.0, a2=1.0))
    if not he["feasible"]:
        return
    b = brute_helr(t.replace(a1=0.0, a2=1.0))
    assert len(he["devices"]) == len(b[1])                       # S:399 minimal subset size
    # adding a device never increases the optimal objective
    r5 = oracle.helr(t)
    extra = W.random_topology(seed + 1000, 6)
    D = 6
    mem = np.concatenate([t.memory_bytes, extra.memory_bytes[:1]])
    perf = np.concatenate([t.performance, extra.performance[:1]])
    lat = np.zeros((D, D))
    lat[:5, :5] = t.link_latency_s
    lat[5, :5] = lat[:5, 5] = extra.link_latency_s[0, 1:]
    r6 = oracle.helr(t.replace(memory_bytes=mem, performance=perf, link_latency_s=lat))
    assert r6["objective"] <= r5["objective"]


def test_cluster_topology_runs():
    r = oracle.helr(W.b200_cluster(nodes=1, per_node=8))
    assert r["feasible"] and sum(r["layer_count"]) == 80


# ---------------------------------------------------------------------------- BGS (O13)
def test_spec_s391_s393_bgs():
    # memories {20, 10} layer-units for 25 layers -> [(d0, 0..19), (d1, 20..24)]
    t = W.Topology(np.array([20, 10], np.uint64), np.array([1.0, 1.0]), np.array([[0, 1.0], [1.0, 0]]),
                   num_layers=25, model_bytes=25)
    r = oracle.bgs(t)
    assert r["devices"] == [0, 1] and r["layer_begin"] == [0, 20] and r["layer_count"] == [20, 5]
    # all layers fit on the largest device -> singleton
    r = oracle.bgs(t.replace(memory_bytes=np.array([10, 30], np.uint64)))
    assert r["devices"] == [1] and r["layer_count"] == [25]
    # equal memories -> tie broken by device id
    r = oracle.bgs(t.replace(memory_bytes=np.array([15, 15], np.uint64)))
    assert r["devices"] == [0, 1] and r["layer_count"] == [15, 10]
    # infeasible
    assert not oracle.bgs(t.replace(memory_bytes=np.array([5, 5], np.uint64)))["feasible"]


@pytest.mark.parametrize("seed", range(60))
def test_bgs_never_beats_helr(seed):
    # BGS's chain is one of the chains HELR searches (same greedy fill, same cost arithmetic)
    t = W.random_topology(seed, 1 + seed % 7)
    b, h = oracle.bgs(t), oracle.helr(t)
    assert b["feasible"] == h["feasible"]
    if b["feasible"]:
        assert h["objective"] <= b["objective"]
        assert chain_latency(t, b["devices"]) == b["latency_s"]
        assert sum(b["layer_count"]) == t.num_layers
        mem = [int(t.memory_bytes[d]) for d in b["devices"]]
        assert mem == sorted(mem, reverse=True)
