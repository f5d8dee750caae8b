"""ctypes binding of the CPU oracle (oracle/uellm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by paper_2409_14961_b200/.

parity pins: see oracle/uellm_oracle.c header and DESIGN.md "Oracle and its pins".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "uellm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_CONTRACT", 3: "ERR_CONFIG", 4: "ERR_OVERFLOW"}


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS.get(status, status)}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11 + pthreads, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-pthread", "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class OrcConfig(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("window", C.c_uint32), ("max_batch", C.c_uint32),
                ("split_on_slo_change", C.c_uint32), ("kv_bytes_per_elem", C.c_uint32),
                ("n_layers", C.c_uint32), ("hidden", C.c_uint32), ("pad0", C.c_uint32),
                ("kv_cap_bytes", C.c_uint64),
                ("t_batch_us", C.c_uint32), ("t_iter_us", C.c_uint32), ("t_tok_us", C.c_uint32),
                ("t_prefill_us", C.c_uint32), ("lambda_us", C.c_uint64),
                ("w1", C.c_double), ("w2", C.c_double), ("l1", C.c_double), ("l2", C.c_double),
                ("threshold", C.c_double), ("eps", C.c_double),
                ("eq2_additive", C.c_uint32), ("pad1", C.c_uint32)]


BATCH_STAT_DTYPE = np.dtype([
    ("start", "<u4"), ("size", "<u4"), ("max_in", "<u4"), ("max_out", "<u4"),
    ("gen_tokens", "<u8"), ("pad_in", "<u8"), ("pad_out", "<u8"), ("kv_bytes", "<u8"),
    ("est_us", "<u8"), ("completion_us", "<u8"),
    ("viol_alone", "<u4"), ("viol_seq", "<u4"), ("over_cap", "<u4"), ("window", "<u4")])


class OrcTotals(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n", "batches", "gen_tokens", "pad_in", "pad_out",
                                          "kv_bytes_max", "dp_cost", "viol_alone", "viol_seq",
                                          "over_cap", "makespan_us")] + \
               [("mean_latency_s", C.c_double), ("throughput_tok_s", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class OrcSimTotals(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n", "batches", "makespan_us", "busy_us", "idle_us",
                                          "gen_tokens", "viol", "latency_max_us",
                                          "latency_sum_lo", "latency_sum_hi")] + \
               [(k, C.c_double) for k in ("mean_latency_s", "slo_violation_rate", "utilization",
                                          "throughput_tok_s")]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["latency_sum_us"] = d["latency_sum_lo"] + (d["latency_sum_hi"] << 64)
        return d


class OrcPredictor(C.Structure):
    _fields_ = [("variant", C.c_uint32), ("bucket_width", C.c_uint32), ("constant_tokens", C.c_uint32),
                ("window", C.c_uint32), ("error_rate", C.c_double), ("gamma", C.c_double),
                ("cap", C.c_double), ("seed", C.c_uint64), ("monitor", C.c_uint32), ("pad", C.c_uint32)]


class OrcHelrCfg(C.Structure):
    _fields_ = [("num_devices", C.c_uint32), ("num_layers", C.c_uint32), ("model_bytes", C.c_uint64),
                ("kv_reserve_bytes", C.c_uint64), ("p", C.c_double), ("a1", C.c_double), ("a2", C.c_double)]


class OrcDeviceMap(C.Structure):
    _fields_ = [("count", C.c_uint32), ("feasible", C.c_uint32), ("mask", C.c_uint32), ("pad", C.c_uint32),
                ("device", C.c_uint32 * 32), ("layer_begin", C.c_uint32 * 32), ("layer_count", C.c_uint32 * 32),
                ("objective", C.c_double), ("latency_s", C.c_double)]

    def as_dict(self):
        k = self.count
        return {"feasible": bool(self.feasible), "mask": self.mask, "devices": list(self.device[:k]),
                "layer_begin": list(self.layer_begin[:k]), "layer_count": list(self.layer_count[:k]),
                "objective": self.objective, "latency_s": self.latency_s}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        _lib.orc_slo_us.argtypes = [C.c_float, C.POINTER(C.c_uint32)]
        _lib.orc_kv_bytes.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        _lib.orc_schedule.argtypes = [C.c_uint64, u32p, u32p, f32p, C.POINTER(OrcConfig),
                                      u32p, u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                      C.c_int]
        _lib.orc_stats.argtypes = [C.c_uint64, u32p, u32p, f32p, C.POINTER(OrcConfig),
                                   u32p, u32p, C.c_uint64, C.c_void_p, C.POINTER(OrcTotals)]
        u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
        _lib.orc_simulate.argtypes = [C.c_uint64, u32p, u32p, f32p, C.POINTER(OrcConfig),
                                      u32p, u32p, C.c_uint64, u64p, C.c_void_p, C.c_void_p,
                                      C.POINTER(OrcSimTotals)]
        _lib.orc_predict.argtypes = [C.c_uint64, C.c_uint64, u32p, C.POINTER(OrcPredictor), C.c_double, u32p]
        _lib.orc_monitor_observe.argtypes = [C.c_uint64, u32p, u32p, C.c_double, C.c_double,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        _lib.orc_profile_stream.argtypes = [C.c_uint64, u32p, C.POINTER(OrcPredictor), C.c_double, u32p, f64p,
                                            C.POINTER(C.c_uint64)]
        u64p_ = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
        f64p_ = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        _lib.orc_helr.argtypes = [C.POINTER(OrcHelrCfg), u64p_, f64p_, f64p_, C.POINTER(OrcDeviceMap)]
        _lib.orc_bgs.argtypes = [C.POINTER(OrcHelrCfg), u64p_, f64p_, f64p_, C.POINTER(OrcDeviceMap)]
        for f in ("orc_sizeof_config", "orc_sizeof_batch_stat", "orc_sizeof_totals",
                  "orc_sizeof_sim_totals", "orc_sizeof_predictor", "orc_sizeof_device_map"):
            getattr(_lib, f).restype = C.c_uint64
        assert _lib.orc_sizeof_config() == C.sizeof(OrcConfig)
        assert _lib.orc_sizeof_batch_stat() == BATCH_STAT_DTYPE.itemsize
        assert _lib.orc_sizeof_totals() == C.sizeof(OrcTotals)
        assert _lib.orc_sizeof_sim_totals() == C.sizeof(OrcSimTotals)
        assert _lib.orc_sizeof_predictor() == C.sizeof(OrcPredictor)
        assert _lib.orc_sizeof_device_map() == C.sizeof(OrcDeviceMap)
    return _lib


def to_config(cfg) -> OrcConfig:
    c = OrcConfig()
    for name, _ in OrcConfig._fields_:
        if name.startswith("pad"):
            continue
        setattr(c, name, getattr(cfg, name))
    return c


def slo_us(x: float) -> int:
    v = C.c_uint32()
    st = lib().orc_slo_us(C.c_float(x), C.byref(v))
    if st:
        raise OracleError(st, "slo_us")
    return v.value


def kv_bytes(kvpe, b, l, h, s, n) -> int:
    v = C.c_uint64()
    st = lib().orc_kv_bytes(kvpe, b, l, h, s, n, C.byref(v))
    if st:
        raise OracleError(st, "kv_bytes")
    return v.value


def _arrays(inp, out, slo):
    return (np.ascontiguousarray(inp, np.uint32), np.ascontiguousarray(out, np.uint32),
            np.ascontiguousarray(slo, np.float32))


def schedule(inp, out, slo, cfg, nthreads: int = 1):
    """-> (order u32[n], offsets u32[m+1], m, dp_cost)."""
    inp, out, slo = _arrays(inp, out, slo)
    n = inp.shape[0]
    order = np.zeros(max(n, 1), np.uint32)
    offsets = np.zeros(n + 1, np.uint32)
    m = C.c_uint64()
    cost = C.c_uint64()
    c = to_config(cfg)
    st = lib().orc_schedule(n, inp, out, slo, C.byref(c), order, offsets, C.byref(m),
                            C.byref(cost), nthreads)
    if st:
        raise OracleError(st, "schedule")
    return order[:n], offsets[: m.value + 1], m.value, cost.value


def stats(inp, out, slo, cfg, order, offsets):
    """-> (per_batch structured array, totals dict)."""
    inp, out, slo = _arrays(inp, out, slo)
    n = inp.shape[0]
    order = np.ascontiguousarray(order, np.uint32)
    offsets = np.ascontiguousarray(offsets, np.uint32)
    m = offsets.shape[0] - 1
    pb = np.zeros(max(m, 1), BATCH_STAT_DTYPE)
    tot = OrcTotals()
    c = to_config(cfg)
    if n == 0:
        order = np.zeros(1, np.uint32)
        inp = out = np.zeros(1, np.uint32)
        slo = np.zeros(1, np.float32)
    st = lib().orc_stats(n, inp, out, slo, C.byref(c), order, offsets, m,
                         pb.ctypes.data_as(C.c_void_p), C.byref(tot))
    if st:
        raise OracleError(st, "stats")
    return pb[:m], tot.as_dict()


def simulate(inp, out, slo, cfg, order, offsets, arrival_us):
    """O8 (NEXT f2): sequential execution with arrivals -> (batch_end u64[m], latency u64[n]
    in scheduled order (latency[k] belongs to query order[k]), totals dict)."""
    inp, out, slo = _arrays(inp, out, slo)
    n = inp.shape[0]
    order = np.ascontiguousarray(order, np.uint32)
    offsets = np.ascontiguousarray(offsets, np.uint32)
    arr = np.ascontiguousarray(arrival_us, np.uint64)
    m = offsets.shape[0] - 1
    ends = np.zeros(max(m, 1), np.uint64)
    lat = np.zeros(max(n, 1), np.uint64)
    tot = OrcSimTotals()
    c = to_config(cfg)
    if n == 0:
        order = np.zeros(1, np.uint32)
        inp = out = np.zeros(1, np.uint32)
        slo = np.zeros(1, np.float32)
        arr = np.zeros(1, np.uint64)
    st = lib().orc_simulate(n, inp, out, slo, C.byref(c), order, offsets, m, arr,
                            ends.ctypes.data_as(C.c_void_p), lat.ctypes.data_as(C.c_void_p),
                            C.byref(tot))
    if st:
        raise OracleError(st, "simulate")
    return ends[:m], lat[:n], tot.as_dict()


PREDICTORS = {"oracle": 0, "bucketed": 1, "noisy": 2, "constant": 3}


def to_predictor(pc) -> OrcPredictor:
    p = OrcPredictor()
    for name, _ in OrcPredictor._fields_:
        if name != "pad":
            setattr(p, name, getattr(pc, name))
    return p


def predict(true_len, pc, factor: float = 1.0, index0: int = 0):
    """O9 (NEXT f4): predicted output lengths of queries index0.. with inflation `factor`."""
    t = np.ascontiguousarray(true_len, np.uint32)
    pred = np.zeros(max(len(t), 1), np.uint32)
    st = lib().orc_predict(len(t), index0, t if len(t) else np.zeros(1, np.uint32), C.byref(to_predictor(pc)),
                           factor, pred)
    if st:
        raise OracleError(st, "predict")
    return pred[: len(t)]


def monitor_observe(pred, actual, gamma: float, cap: float, corrections: int = 0, factor: float = 1.0):
    """O10 (NEXT f4): -> (corrections, factor) after observing every (pred, actual) in order."""
    p = np.ascontiguousarray(pred, np.uint32)
    a = np.ascontiguousarray(actual, np.uint32)
    c = C.c_uint64(corrections)
    f = C.c_double(factor)
    st = lib().orc_monitor_observe(len(p), p if len(p) else np.zeros(1, np.uint32),
                                   a if len(a) else np.zeros(1, np.uint32), gamma, cap, C.byref(c), C.byref(f))
    if st:
        raise OracleError(st, "monitor_observe")
    return c.value, f.value


def profile_stream(true_len, pc, factor0: float = 1.0):
    """O11 (NEXT f4, R20): -> (pred u32[n], factors f64[nwin + 1], corrections)."""
    t = np.ascontiguousarray(true_len, np.uint32)
    n = len(t)
    wl = pc.window or max(n, 1)
    nwin = (n + wl - 1) // wl
    pred = np.zeros(max(n, 1), np.uint32)
    factors = np.zeros(nwin + 1, np.float64)
    c = C.c_uint64()
    st = lib().orc_profile_stream(n, t if n else np.zeros(1, np.uint32), C.byref(to_predictor(pc)), factor0, pred,
                                  factors, C.byref(c))
    if st:
        raise OracleError(st, "profile_stream")
    return pred[:n], factors, c.value


def helr(topo):
    """O12 (NEXT f3): HELR device map of a workloads.Topology -> dict."""
    c = OrcHelrCfg(len(topo.memory_bytes), topo.num_layers, topo.model_bytes, topo.kv_reserve_bytes,
                   topo.p, topo.a1, topo.a2)
    mem = np.ascontiguousarray(topo.memory_bytes, np.uint64)
    perf = np.ascontiguousarray(topo.performance, np.float64)
    lat = np.ascontiguousarray(topo.link_latency_s, np.float64).reshape(-1)
    out = OrcDeviceMap()
    st = lib().orc_helr(C.byref(c), mem, perf, lat, C.byref(out))
    if st:
        raise OracleError(st, "helr")
    return out.as_dict()


def bgs(topo):
    """O13 (NEXT f3): the BGS baseline deployer's device map of a workloads.Topology -> dict."""
    c = OrcHelrCfg(len(topo.memory_bytes), topo.num_layers, topo.model_bytes, topo.kv_reserve_bytes,
                   topo.p, topo.a1, topo.a2)
    mem = np.ascontiguousarray(topo.memory_bytes, np.uint64)
    perf = np.ascontiguousarray(topo.performance, np.float64)
    lat = np.ascontiguousarray(topo.link_latency_s, np.float64).reshape(-1)
    out = OrcDeviceMap()
    st = lib().orc_bgs(C.byref(c), mem, perf, lat, C.byref(out))
    if st:
        raise OracleError(st, "bgs")
    return out.as_dict()
