"""Thin ctypes binding of libuellm.so (include/uellm.h).  Argument marshalling only: every
step of the scheduling path runs in the library's sm_100a kernels.  PyTorch supplies device
memory (workspace and outputs) and streams; numpy / pinned host arrays may be passed where the
header allows [host|device] pointers.

There is no fallback: if libuellm.so is missing or fails to load, importing this module
raises.  Names mirror the C ABI (uellm_profile_load -> profile_load, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libuellm.so")

OK, ERR_ARG, ERR_CONTRACT, ERR_CONFIG, ERR_OVERFLOW, ERR_CUDA, ERR_UNSUPPORTED, ERR_STALE = range(8)
MODE_SEG_DP, MODE_SLO_ODBS, MODE_FIFO, MODE_SORT_ONLY = range(4)


class UellmError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("window", C.c_uint32), ("max_batch", C.c_uint32),
                ("split_on_slo_change", C.c_uint32), ("kv_bytes_per_elem", C.c_uint32),
                ("n_layers", C.c_uint32), ("hidden", C.c_uint32), ("dp_tile", C.c_uint32),
                ("kv_cap_bytes", C.c_uint64),
                ("t_batch_us", C.c_uint32), ("t_iter_us", C.c_uint32), ("t_tok_us", C.c_uint32),
                ("t_prefill_us", C.c_uint32), ("lambda_us", C.c_uint64),
                ("w1", C.c_double), ("w2", C.c_double), ("l1", C.c_double), ("l2", C.c_double),
                ("threshold", C.c_double), ("eps", C.c_double),
                ("eq2_additive", C.c_uint32), ("flags", C.c_uint32)]


class Queries(C.Structure):
    _fields_ = [("n", C.c_uint64), ("input_len", C.c_void_p), ("pred_out_len", C.c_void_p),
                ("slo_s", C.c_void_p)]


class Totals(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n", "batches", "gen_tokens", "pad_in", "pad_out",
                                          "kv_bytes_max", "dp_cost", "viol_alone", "viol_seq",
                                          "over_cap", "makespan_us")] + \
               [("mean_latency_s", C.c_double), ("throughput_tok_s", C.c_double),
                ("latency_sum_lo", C.c_uint64), ("latency_sum_hi", C.c_uint64), ("overflow", C.c_uint64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["latency_sum_us"] = d["latency_sum_lo"] + (d["latency_sum_hi"] << 64)
        return d


class SimTotals(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n", "batches", "makespan_us", "busy_us", "idle_us",
                                          "gen_tokens", "viol", "latency_max_us",
                                          "latency_sum_lo", "latency_sum_hi")] + \
               [(k, C.c_double) for k in ("mean_latency_s", "slo_violation_rate", "utilization",
                                          "throughput_tok_s")] + \
               [("status", C.c_uint32), ("pad", C.c_uint32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}
        d["latency_sum_us"] = d["latency_sum_lo"] + (d["latency_sum_hi"] << 64)
        return d


class Predictor(C.Structure):
    _fields_ = [("variant", C.c_uint32), ("bucket_width", C.c_uint32), ("constant_tokens", C.c_uint32),
                ("window", C.c_uint32), ("error_rate", C.c_double), ("gamma", C.c_double),
                ("cap", C.c_double), ("seed", C.c_uint64), ("monitor", C.c_uint32), ("pad", C.c_uint32)]


class MonitorState(C.Structure):
    _fields_ = [("corrections", C.c_uint64), ("inflation_factor", C.c_double), ("scratch", C.c_uint64 * 2)]


class Topology(C.Structure):
    _fields_ = [("num_devices", C.c_uint32), ("num_layers", C.c_uint32), ("model_bytes", C.c_uint64),
                ("kv_reserve_bytes", C.c_uint64), ("p", C.c_double), ("a1", C.c_double), ("a2", C.c_double),
                ("memory_bytes", C.c_void_p), ("performance", C.c_void_p), ("link_latency_s", C.c_void_p)]


class DeviceMap(C.Structure):
    _fields_ = [("count", C.c_uint32), ("feasible", C.c_uint32), ("mask", C.c_uint32), ("pad", C.c_uint32),
                ("device", C.c_uint32 * 32), ("layer_begin", C.c_uint32 * 32), ("layer_count", C.c_uint32 * 32),
                ("objective", C.c_double), ("latency_s", C.c_double)]

    def as_dict(self):
        k = self.count
        return {"feasible": bool(self.feasible), "mask": self.mask, "devices": list(self.device[:k]),
                "layer_begin": list(self.layer_begin[:k]), "layer_count": list(self.layer_count[:k]),
                "objective": self.objective, "latency_s": self.latency_s}


class Profile(C.Structure):
    _fields_ = [("opaque", C.c_uint64 * 40)]


def p_n(p: "Profile") -> int:
    """Query count of a loaded profile (second word of the opaque view)."""
    return int(p.opaque[1])


class Diagnostics(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("tiles", "tile_len", "fixups_unconverged", "cascade_reruns",
                                          "fixup_positions", "trace_unmerged", "trace_rewalks",
                                          "sort_passes", "dp_cost", "dp_candidate_evals",
                                          "sched_launches", "stats_launches", "sort_key_bits",
                                          "dp_filled_positions")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


BATCH_STAT_DTYPE = np.dtype([
    ("start", "<u4"), ("size", "<u4"), ("max_in", "<u4"), ("max_out", "<u4"),
    ("gen_tokens", "<u8"), ("pad_in", "<u8"), ("pad_out", "<u8"), ("kv_bytes", "<u8"),
    ("est_us", "<u8"), ("completion_us", "<u8"),
    ("viol_alone", "<u4"), ("viol_seq", "<u4"), ("over_cap", "<u4"), ("window", "<u4")])
TOTALS_BYTES = C.sizeof(Totals)
SIM_TOTALS_BYTES = C.sizeof(SimTotals)

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libuellm.so not built ({_LIB_PATH}); run __graft_entry__.build()")
_lib = C.CDLL(_LIB_PATH)
_lib.uellm_abi_version.restype = C.c_uint32
_lib.uellm_sizeof.restype = C.c_uint64
_lib.uellm_sizeof.argtypes = [C.c_int]
_lib.uellm_status_string.restype = C.c_char_p
_lib.uellm_status_string.argtypes = [C.c_int32]
_lib.uellm_workspace_bytes.restype = C.c_size_t
_lib.uellm_workspace_bytes.argtypes = [C.c_uint64, C.POINTER(Config)]
_lib.uellm_profile_load.restype = C.c_int32
_lib.uellm_profile_load.argtypes = [C.POINTER(Queries), C.POINTER(Config), C.c_void_p, C.c_size_t,
                                    C.c_void_p, C.POINTER(Profile)]
_lib.uellm_profile_reload.restype = C.c_int32
_lib.uellm_profile_reload.argtypes = [C.POINTER(Profile), C.POINTER(Queries), C.POINTER(Config), C.c_void_p]
_lib.uellm_profile_status.restype = C.c_int32
_lib.uellm_profile_status.argtypes = [C.POINTER(Profile), C.POINTER(C.c_void_p)]
_lib.uellm_schedule_batches.restype = C.c_int32
_lib.uellm_schedule_batches.argtypes = [C.POINTER(Profile), C.POINTER(Config), C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
_lib.uellm_batch_stats.restype = C.c_int32
_lib.uellm_batch_stats.argtypes = [C.POINTER(Profile), C.POINTER(Config), C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
_lib.uellm_simulate.restype = C.c_int32
_lib.uellm_simulate.argtypes = [C.POINTER(Profile), C.POINTER(Config)] + [C.c_void_p] * 8
_lib.uellm_predict_lengths.restype = C.c_int32
_lib.uellm_predict_lengths.argtypes = [C.c_uint64, C.c_void_p, C.POINTER(Predictor)] + [C.c_void_p] * 3 + \
    [C.c_void_p, C.c_size_t, C.c_void_p]
_lib.uellm_predict_workspace_bytes.restype = C.c_size_t
_lib.uellm_predict_workspace_bytes.argtypes = [C.c_uint64, C.POINTER(Predictor)]
_lib.uellm_helr_workspace_bytes.restype = C.c_size_t
_lib.uellm_helr_workspace_bytes.argtypes = [C.c_uint32]
_lib.uellm_helr_plan.restype = C.c_int32
_lib.uellm_helr_plan.argtypes = [C.POINTER(Topology), C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
_lib.uellm_bgs_plan.restype = C.c_int32
_lib.uellm_bgs_plan.argtypes = [C.POINTER(Topology), C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
_lib.uellm_boundary_bitmap.restype = C.c_int32
_lib.uellm_boundary_bitmap.argtypes = [C.POINTER(Profile), C.POINTER(Config), C.c_void_p, C.c_void_p]
_lib.uellm_pipeline_workspace_bytes.restype = C.c_size_t
_lib.uellm_pipeline_workspace_bytes.argtypes = [C.c_uint64, C.POINTER(Config), C.c_uint32]
_lib.uellm_schedule_pipelined.restype = C.c_int32
_lib.uellm_schedule_pipelined.argtypes = [C.POINTER(Queries), C.POINTER(Config), C.c_uint32, C.c_void_p,
                                          C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_lib.uellm_exchange_bytes.restype = C.c_size_t
_lib.uellm_exchange_bytes.argtypes = [C.c_uint64]
_lib.uellm_exchange_pack.restype = C.c_int32
_lib.uellm_exchange_pack.argtypes = [C.POINTER(Profile), C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_uint64,
                                     C.c_void_p]
_lib.uellm_exchange_workspace_bytes.restype = C.c_size_t
_lib.uellm_exchange_workspace_bytes.argtypes = [C.c_uint64, C.c_uint32]
_lib.uellm_exchange_combine.restype = C.c_int32
_lib.uellm_exchange_combine.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_size_t,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_lib.uellm_totals_combine.restype = C.c_int32
_lib.uellm_totals_combine.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_size_t,
                                      C.c_void_p]
_lib.uellm_set_stage_events.restype = C.c_int32
_lib.uellm_set_stage_events.argtypes = [C.POINTER(Profile), C.POINTER(C.c_void_p), C.c_uint32]
_lib.uellm_get_diagnostics.restype = C.c_int32
_lib.uellm_get_diagnostics.argtypes = [C.POINTER(Profile), C.POINTER(Diagnostics), C.c_void_p]

assert _lib.uellm_abi_version() == 3
assert _lib.uellm_sizeof(0) == C.sizeof(Config)
assert _lib.uellm_sizeof(1) == BATCH_STAT_DTYPE.itemsize == 80
assert _lib.uellm_sizeof(2) == C.sizeof(Totals)
assert _lib.uellm_sizeof(3) == C.sizeof(Profile)
assert _lib.uellm_sizeof(4) == C.sizeof(Diagnostics)
assert _lib.uellm_sizeof(5) == C.sizeof(SimTotals)
assert _lib.uellm_sizeof(6) == C.sizeof(Predictor)
assert _lib.uellm_sizeof(7) == C.sizeof(MonitorState)
assert _lib.uellm_sizeof(8) == C.sizeof(Topology)
assert _lib.uellm_sizeof(9) == C.sizeof(DeviceMap)

LIBRARY_PATH = _LIB_PATH


def status_string(s: int) -> str:
    return _lib.uellm_status_string(s).decode()


def _check(st: int, what: str):
    if st != OK:
        raise UellmError(st, what)


def make_config(cfg) -> Config:
    """Build the C config from any object with the uellm_config field names (e.g.
    workloads.SchedConfig)."""
    c = Config()
    for name, _ in Config._fields_:
        if hasattr(cfg, name):
            setattr(c, name, getattr(cfg, name))
    return c


def _ptr(x) -> int | None:
    """Raw address of a torch tensor / numpy array (no copies: marshalling only)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    return int(x)


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def workspace_bytes(n: int, cfg: Config) -> int:
    return _lib.uellm_workspace_bytes(n, C.byref(cfg))


def profile_load(n: int, input_len, pred_out_len, slo_s, cfg: Config, ws, ws_bytes: int,
                 stream=None) -> Profile:
    q = Queries(n, _ptr(input_len), _ptr(pred_out_len), _ptr(slo_s))
    p = Profile()
    _check(_lib.uellm_profile_load(C.byref(q), C.byref(cfg), _ptr(ws), ws_bytes,
                                   _stream_handle(stream), C.byref(p)), "uellm_profile_load")
    return p


def profile_reload(p: Profile, input_len, pred_out_len, slo_s, cfg: Config, stream=None) -> Profile:
    """Asynchronous re-load of the next queries (device arrays) into `p` (updated in place); the
    verdict goes to the device status word (profile_status)."""
    q = Queries(p_n(p), _ptr(input_len), _ptr(pred_out_len), _ptr(slo_s))
    _check(_lib.uellm_profile_reload(C.byref(p), C.byref(q), C.byref(cfg), _stream_handle(stream)),
           "uellm_profile_reload")
    return p


def profile_status(p: Profile) -> int:
    """Device address of the profile's u32 status word."""
    w = C.c_void_p()
    _check(_lib.uellm_profile_status(C.byref(p), C.byref(w)), "uellm_profile_status")
    return w.value


def schedule_batches(p: Profile, cfg: Config, order, batch_offsets, num_batches, stream=None):
    _check(_lib.uellm_schedule_batches(C.byref(p), C.byref(cfg), _ptr(order), _ptr(batch_offsets),
                                       _ptr(num_batches), _stream_handle(stream)),
           "uellm_schedule_batches")


def batch_stats(p: Profile, cfg: Config, batch_offsets, num_batches, per_batch, totals, stream=None):
    _check(_lib.uellm_batch_stats(C.byref(p), C.byref(cfg), _ptr(batch_offsets), _ptr(num_batches),
                                  _ptr(per_batch), _ptr(totals), _stream_handle(stream)),
           "uellm_batch_stats")


def simulate(p: Profile, cfg: Config, arrival_us, order, batch_offsets, num_batches, batch_end_us,
             latency_us, totals, stream=None):
    _check(_lib.uellm_simulate(C.byref(p), C.byref(cfg), _ptr(arrival_us), _ptr(order), _ptr(batch_offsets),
                               _ptr(num_batches), _ptr(batch_end_us), _ptr(latency_us), _ptr(totals),
                               _stream_handle(stream)), "uellm_simulate")


def make_predictor(pc) -> Predictor:
    """C predictor from any object with the uellm_predictor field names (workloads.PredictorConfig)."""
    p = Predictor()
    for name, _ in Predictor._fields_:
        if name != "pad" and hasattr(pc, name):
            setattr(p, name, getattr(pc, name))
    return p


def predict_workspace_bytes(n: int, pc: Predictor) -> int:
    return _lib.uellm_predict_workspace_bytes(n, C.byref(pc))


def predict_lengths(n: int, true_out_len, pc: Predictor, state, pred_out_len, window_factors=None, stream=None,
                    ws=None, ws_bytes: int = 0):
    _check(_lib.uellm_predict_lengths(n, _ptr(true_out_len), C.byref(pc), _ptr(state), _ptr(pred_out_len),
                                      _ptr(window_factors), _ptr(ws), ws_bytes, _stream_handle(stream)),
           "uellm_predict_lengths")


def pipeline_workspace_bytes(n: int, cfg: Config, groups: int = 0) -> int:
    return _lib.uellm_pipeline_workspace_bytes(n, C.byref(cfg), groups)


def schedule_pipelined(n: int, input_len, pred_out_len, slo_s, cfg: Config, groups: int, ws, ws_bytes: int,
                       order, batch_offsets, num_batches, totals, stream=None):
    q = Queries(n, _ptr(input_len), _ptr(pred_out_len), _ptr(slo_s))
    _check(_lib.uellm_schedule_pipelined(C.byref(q), C.byref(cfg), groups, _ptr(ws), ws_bytes, _ptr(order),
                                         _ptr(batch_offsets), _ptr(num_batches), _ptr(totals),
                                         _stream_handle(stream)), "uellm_schedule_pipelined")


def boundary_bitmap(p: Profile, cfg: Config, words, stream=None):
    _check(_lib.uellm_boundary_bitmap(C.byref(p), C.byref(cfg), _ptr(words), _stream_handle(stream)),
           "uellm_boundary_bitmap")


def exchange_bytes(n_max: int) -> int:
    return _lib.uellm_exchange_bytes(n_max)


def exchange_pack(p: Profile, cfg: Config, totals, record, n_max: int, stream=None):
    _check(_lib.uellm_exchange_pack(C.byref(p), C.byref(cfg), _ptr(totals), _ptr(record), n_max,
                                    _stream_handle(stream)), "uellm_exchange_pack")


def totals_combine(parts, count: int, stride_bytes: int, out, ws=None, ws_bytes: int = 0, stream=None):
    _check(_lib.uellm_totals_combine(_ptr(parts), count, stride_bytes, _ptr(out), _ptr(ws), ws_bytes,
                                     _stream_handle(stream)), "uellm_totals_combine")


def exchange_workspace_bytes(n_total: int, world: int) -> int:
    return _lib.uellm_exchange_workspace_bytes(n_total, world)


def exchange_combine(gathered, world: int, n_max: int, query_begin, ws, ws_bytes: int, batch_offsets, num_batches,
                     totals, stream=None):
    qb = np.ascontiguousarray(query_begin, np.uint64)
    if qb.shape != (world + 1,):
        raise ValueError("query_begin needs world + 1 entries")
    _check(_lib.uellm_exchange_combine(_ptr(gathered), world, n_max, qb.ctypes.data, _ptr(ws), ws_bytes,
                                       _ptr(batch_offsets), _ptr(num_batches), _ptr(totals), _stream_handle(stream)),
           "uellm_exchange_combine")


def helr_workspace_bytes(num_devices: int) -> int:
    return _lib.uellm_helr_workspace_bytes(num_devices)


def _topology(topo):
    mem = np.ascontiguousarray(topo.memory_bytes, np.uint64)
    perf = np.ascontiguousarray(topo.performance, np.float64)
    lat = np.ascontiguousarray(topo.link_latency_s, np.float64)
    t = Topology(len(mem), topo.num_layers, topo.model_bytes, topo.kv_reserve_bytes, topo.p, topo.a1, topo.a2,
                 mem.ctypes.data, perf.ctypes.data, lat.ctypes.data)
    return t, (mem, perf, lat)


def bgs_plan(topo, ws, ws_bytes: int, out=None, stream=None) -> DeviceMap | None:
    """The BGS baseline deployer (same arguments as helr_plan)."""
    t, keep = _topology(topo)
    host = DeviceMap() if out is None else None
    _check(_lib.uellm_bgs_plan(C.byref(t), _ptr(ws), ws_bytes, C.addressof(host) if host is not None else _ptr(out),
                               _stream_handle(stream)), "uellm_bgs_plan")
    del keep
    return host


def helr_plan(topo, ws, ws_bytes: int, out=None, stream=None) -> DeviceMap | None:
    """topo: any object with the uellm_topology scalar fields + numpy arrays memory_bytes (u64),
    performance (f64), link_latency_s (f64 [D, D]) (e.g. workloads.Topology).  out=None returns a
    host DeviceMap (synchronising); otherwise out is a device buffer of sizeof(DeviceMap) bytes."""
    mem = np.ascontiguousarray(topo.memory_bytes, np.uint64)
    perf = np.ascontiguousarray(topo.performance, np.float64)
    lat = np.ascontiguousarray(topo.link_latency_s, np.float64)
    t = Topology(len(mem), topo.num_layers, topo.model_bytes, topo.kv_reserve_bytes, topo.p, topo.a1, topo.a2,
                 mem.ctypes.data, perf.ctypes.data, lat.ctypes.data)
    host = DeviceMap() if out is None else None
    _check(_lib.uellm_helr_plan(C.byref(t), _ptr(ws), ws_bytes, C.addressof(host) if host is not None else _ptr(out),
                                _stream_handle(stream)), "uellm_helr_plan")
    return host


STAGES = ["sched_begin", "sort_end", "decode_end", "dp_local_end", "dp_fix_end", "dp_cascade_end",
          "trace_end", "sched_end", "stats_begin", "stats_end"]


def set_stage_events(p: Profile, events):
    """events: sequence of torch.cuda.Event(enable_timing=True) (or raw handles / None)."""
    arr = (C.c_void_p * max(len(events), 1))(*[None if e is None else
                                               (e.cuda_event if hasattr(e, "cuda_event") else int(e))
                                               for e in events])
    _check(_lib.uellm_set_stage_events(C.byref(p), arr, len(events)), "uellm_set_stage_events")


def get_diagnostics(p: Profile, stream=None) -> dict:
    d = Diagnostics()
    _check(_lib.uellm_get_diagnostics(C.byref(p), C.byref(d), _stream_handle(stream)),
           "uellm_get_diagnostics")
    return d.as_dict()
