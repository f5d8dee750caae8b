#!/usr/bin/env python
"""Benchmark of the UELLM batch-scheduler hot path on B200 (BASELINE.json metric:
"queries scheduled/sec (device-timed, max over ranks) and HBM GB/s vs roofline").

One step = one pass of the whole hot path over one batch of synthetic queries resident in HBM:
uellm_profile_load (validate + SLO->us + key pack) -> uellm_schedule_batches (radix sort,
SEG-DP, traceback, offsets) -> uellm_batch_stats (per-batch stats + totals), plus, at N > 1,
the a9 exchange (uellm_exchange_pack -> ONE NCCL all_gather_into_tensor -> uellm_exchange_combine,
which rebuilds the whole job's batch_offsets and totals on every rank).  Workload: BJ configs[3]
(c4: ONE job of 10^8 queries in 10^6-query windows), sharded across the N ranks by contiguous
window blocks (strong scaling: value = 10^8 / max-over-ranks step time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl uellm|reference] [--config c4]

--impl reference times the CPU oracle (oracle/, as it stands) on the host cores, on a bounded
sample of the same workload.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "queries scheduled/sec (device-timed, max over ranks)"
UNIT = "queries/s"
# SEG-DP issue roofline: warp instructions per candidate evaluation as
# measured by ncu (fallback if profiles/ncu_summary.json is absent)
DP_WARP_INST_PER_EVAL = 2.064
SMS = 148
ISSUE_PER_SM = 4


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("sm_max_mhz", 1965.0), "measured"
    return 6650.0, 1965.0, "fallback"


def workload(name: str, rank: int, n_override: int | None):
    import workloads as W
    if name == "c4":
        n = n_override or 100_000_000
        inp, out, slo, cfg = W.c4(seed=rank, n=n)
        return "c4: 1e8 queries, 1e6-query windows, 8 SLO classes, long-tail outputs <=4096, " \
               "LLaMA-2-7B KV cap, W=256, lambda=1e9 us", inp, out, slo, cfg
    if name == "c2":
        inp, out, slo, cfg = W.c2(seed=rank, n=n_override or 10_000)
        return "c2: 1e4 queries, one window", inp, out, slo, cfg
    if name == "c3":
        inp, out, slo, cfg = W.c3(seed=rank, n=n_override or 1_000_000)
        return "c3: 1e6 queries, one window", inp, out, slo, cfg
    if name == "c5":
        inp, out, slo, cfg = W.c5(seed=rank, n=n_override or 10_000_000)
        return "c5: 1e7 adversarial queries, 1e6-query windows", inp, out, slo, cfg
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def compulsory_bytes(n: int, m: int) -> int:
    # 12 B/query read (in, out, slo), 4 B/query order, 4 B per offset,
    # 80 B per-batch record, totals
    return 12 * n + 4 * n + 4 * (m + 1) + 80 * m + 112


def ncu_summary() -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, if present."""
    ks = ncu_summary().get("kernels", {})
    # exact name, else the first launch of its instantiation (e.g. k_dp_tiles -> k_dp_tiles<2>)
    k = ks.get(kernel) or next((v for n, v in ks.items() if n.split("<")[0] == kernel and "#" not in n), None)
    return k.get("dram_bytes_per_launch") if k else None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(inp, out, slo, cfg, windows: int):
    """The oracle as it stands on the host cores, on a bounded sample (first `windows` windows),
    plus one window on one thread (core count, CPU model, single-thread run)."""
    import oracle
    cores = os.cpu_count() or 1
    nq = min(len(inp), windows * cfg.window)
    t = time.perf_counter()
    o = oracle.schedule(inp[:nq], out[:nq], slo[:nq], cfg, nthreads=cores)
    oracle.stats(inp[:nq], out[:nq], slo[:nq], cfg, o[0], o[1])
    dt = time.perf_counter() - t
    n1 = min(len(inp), cfg.window or len(inp))
    t = time.perf_counter()
    o = oracle.schedule(inp[:n1], out[:n1], slo[:n1], cfg, nthreads=1)
    oracle.stats(inp[:n1], out[:n1], slo[:n1], cfg, o[0], o[1])
    dt1 = time.perf_counter() - t
    return {"value": nq / dt, "unit": UNIT, "cores": min(cores, windows), "kind": "oracle",
            "cpu_model": cpu_model(), "host_cores": cores,
            "single_thread": {"value": n1 / dt1, "unit": UNIT, "sample": f"first window ({n1} queries), {dt1:.2f} s"},
            "sample": f"first {windows} windows ({nq} queries) of the same workload, schedule + stats, "
                      f"{min(cores, windows)} threads (one window per thread), {dt:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    desc, inp, out, slo, cfg = workload(args.config, 0, args.n)
    cores = os.cpu_count() or 1
    wl = cfg.window or len(inp)
    nwin = max(1, min(cores, len(inp) // wl))
    nq = min(nwin * wl, len(inp))
    import oracle
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        o = oracle.schedule(inp[:nq], out[:nq], slo[:nq], cfg, nthreads=cores)
        oracle.stats(inp[:nq], out[:nq], slo[:nq], cfg, o[0], o[1])
        if it >= args.warmup:
            times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(times))
    value = nq / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": desc, "sample_queries": nq, "windows": nwin},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, nwin), "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{nwin} windows x {wl} queries per step, one window per thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def stage_hbm(st_ms: dict, n: int, m: int, passes: int, hbm_gbs: float, fused: bool = True) -> dict:
    """Per-stage algorithmic bytes / event-timed stage ms / measured HBM peak:
    load 12 B/q read (+ 4 B/q packed keys written by the fused reload of a rank-compressed profile);
    sort: the key pack (12 B/q, unless the reload packed), 8 B/q read + 8 B/q written per radix pass
    (the first pass reads the input length as payload), the last pass writes the 12 B/q records +
    4 B/q order instead; SEG-DP 12 B/q read + 10 B/q written (C, arg); traceback 2 B/q read + n/8
    bitmap; compact n/8 + 4 B/batch; stats 12 B/q + 4 B/batch read, 80 B/batch written."""
    alg = {"load": (16 if fused else 12) * n,
           "sort": 16 * n * passes + 8 * n + (0 if fused else 12 * n),
           "dp": 22 * n,
           "traceback": 2 * n + n // 8,
           "compact": n // 8 + 4 * (m + 1),
           "stats": 12 * n + 84 * m}
    ms = {"load": st_ms["load"], "sort": st_ms["sort"] + st_ms["decode"],
          "dp": st_ms["dp_local"] + st_ms["dp_fix"] + st_ms["dp_cascade"], "traceback": st_ms["traceback"],
          "compact": st_ms["compact"], "stats": st_ms["stats"]}
    out = {}
    for k in alg:
        gbs = alg[k] / (ms[k] / 1e3) / 1e9 if ms[k] > 0 else 0.0
        out[k] = {"ms": ms[k], "algorithmic_bytes": alg[k], "achieved_gbs": gbs, "frac": gbs / hbm_gbs}
    return out


def offsets_digest(offsets: np.ndarray, totals: dict) -> str:
    """sha256 of the job's batch_offsets and integer totals (the N = 1 and N > 1 runs must agree)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(offsets, np.uint32).tobytes())
    for f in ("n", "batches", "gen_tokens", "pad_in", "pad_out", "kv_bytes_max", "dp_cost", "viol_alone",
              "viol_seq", "over_cap", "makespan_us", "latency_sum_us"):
        h.update(str(int(totals[f])).encode())
    return h.hexdigest()


def time_steps(step, K, stream, dev):
    import torch
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(K):
        step(k)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    return t0.elapsed_time(t1) / K


def sub_config(name, K, Wm, stream, dev, hbm_gbs):
    """Another BJ config as a timed sub-record of the same line (N = 1): same step (reload +
    schedule + stats, eager), inputs resident in HBM, CUDA events on the launching stream."""
    import torch
    from paper_2409_14961_b200.scheduler import GpuScheduler
    import workloads as W
    if name == "c2":
        inp, out, slo, cfg = W.c2(0)
        desc = "c2: 1e4 queries, one window, 3 SLO classes, Alpaca-like lengths, W=64"
    elif name == "c3":
        inp, out, slo, cfg = W.c3(0)
        desc = "c3: 1e6 queries, one window, 8 SLO classes, long-tail outputs, W=256"
    else:
        inp, out, slo, cfg = W.c5(0)
        desc = ("c5: 1e7 adversarial queries in 1e6 windows (identical keys, all-violating, 1% over cap, "
                "anti-sorted distinct SLOs), W=256")
    n = len(inp)
    d_in = torch.from_numpy(inp.view(np.int32)).to(dev)
    d_out = torch.from_numpy(out.view(np.int32)).to(dev)
    d_slo = torch.from_numpy(slo).to(dev)
    g = GpuScheduler(n, cfg, device=dev)
    # the same step as the c4 line: one synchronising load first, then reload (device-side
    # validation, no host sync) -> schedule -> stats per step, launched eagerly
    g.load(d_in, d_out, d_slo, stream)

    def step(k=None):
        g.reload(d_in, d_out, d_slo, stream)
        g.schedule(stream)
        g.stats(stream)
    for _ in range(Wm):
        step()
    torch.cuda.synchronize(dev)
    ms = time_steps(step, K, stream, dev)
    if int(g.status_word().item()) != 0:
        raise SystemExit(f"{name}: device status word {int(g.status_word().item())} after the timed steps")
    diag = g.diagnostics(stream)
    res = g.results()
    comp = compulsory_bytes(n, res["m"])
    rec = {"workload": desc, "queries": n, "ms_per_step": ms, "value": n / (ms / 1e3), "unit": UNIT,
           "batches": res["m"], "dp_cost": res["totals"]["dp_cost"],
           "step_hbm_frac": comp / (ms / 1e3) / 1e9 / hbm_gbs,
           "dp_candidate_evals_per_query": diag["dp_candidate_evals"] / max(n, 1),
           "fixups_unconverged": diag["fixups_unconverged"], "cascade_reruns": diag["cascade_reruns"],
           "sort_key_bits": diag["sort_key_bits"]}
    del g
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="uellm", choices=["uellm", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--queries", dest="n", type=int, default=None, help="override query count (testing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sim", action="store_true", help="skip the NEXT-row timings (f1-f4)")
    ap.add_argument("--no-configs", action="store_true", help="skip the c2 / c3 / c5 sub-records")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling extra (N > 1)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo only for multi-rank tests on one GPU)")
    ap.add_argument("--e2e-groups", type=int, default=0, help="window groups of the pipelined e2e call (0 = 12)")
    ap.add_argument("--dp-tile", type=int, default=0, help="SEG-DP tile length override (tuning only)")
    ap.add_argument("--no-graph", action="store_true", help="time the eager step instead of its CUDA graph")
    ap.add_argument("--mode", default="seg_dp", choices=["seg_dp", "slo_odbs", "fifo", "sort_only"],
                    help="segmentation mode (default: the SEG-DP hot path)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200 import distributed as D
    from paper_2409_14961_b200.scheduler import GpuScheduler

    local = local % max(torch.cuda.device_count(), 1)   # (test runs may put several ranks on one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            # the collective's evidence (ranks, NVLink / NVLS transport) goes to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,COLL")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    # ONE job (seed 0), every rank takes its contiguous window block (strong scaling)
    desc, inp_all, out_all, slo_all, cfg = workload(args.config, 0, args.n)
    if args.dp_tile:
        cfg = cfg.replace(dp_tile=args.dp_tile)
    if args.mode != "seg_dp":
        import workloads as W
        cfg = cfg.replace(mode={"slo_odbs": W.MODE_SLO_ODBS, "fifo": W.MODE_FIFO, "sort_only": W.MODE_SORT_ONLY}[args.mode],
                          w1=1.0, w2=0.02, threshold=900.0)
        desc += f"; mode {args.mode} (Alg. 1: w1=1, w2=0.02, threshold=900)" if args.mode == "slo_odbs" else f"; mode {args.mode}"
    n_total = len(inp_all)
    X = D.Exchange(n_total, cfg.window, world, rank, dev) if world > 1 else None
    q0, q1 = (X.q0, X.q1) if X else (0, n_total)
    inp, out, slo = inp_all[q0:q1], out_all[q0:q1], slo_all[q0:q1]
    n = len(inp)
    d_in = torch.from_numpy(inp.view(np.int32)).to(dev)
    d_out = torch.from_numpy(out.view(np.int32)).to(dev)
    d_slo = torch.from_numpy(slo).to(dev)
    stream = torch.cuda.Stream(device=dev)
    g = GpuScheduler(n, cfg, device=dev)
    K, Wm = args.steps, args.warmup
    nst = len(U.STAGES)
    # per-step stage events (caller-owned; recorded by the library on `stream`)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst)] for _ in range(K)]
    ld = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    xe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for row in ev:
            for e in row:
                e.record(stream)          # materialise the cudaEvent_t handles

    def step(k=None, sync_load=False):
        if k is not None:
            ld[k][0].record(stream)
        if sync_load or g.profile is None:
            g.load(d_in, d_out, d_slo, stream)        # validates on the host, fixes the profile's decisions
        else:
            g.reload(d_in, d_out, d_slo, stream)      # same validation on the device, no host sync
        if k is not None:
            ld[k][1].record(stream)
            U.set_stage_events(g.profile, ev[k])
        elif g.profile is not None:
            U.set_stage_events(g.profile, [])
        g.schedule(stream)
        g.stats(stream)
        if X is not None:   # a9: pack -> ONE allgather -> every rank rebuilds the job
            if k is not None:
                xe[k][0].record(stream)
            X.pack(g.profile, g.cfg, g.totals, stream)
            if not local_only:
                exchange(k)

    def exchange(k=None):
        with torch.cuda.stream(stream):
            X.all_gather(backend=args.dist_backend)
        X.combine(stream)
        if k is not None:
            xe[k][1].record(stream)

    local_only = False
    step(sync_load=True)
    for _ in range(Wm - 1):
        step()
    torch.cuda.synchronize(dev)
    # the rank's local step (reload -> schedule -> stats [-> a9 pack]) captured once as a CUDA graph
    # and replayed: one launch, no host synchronisation inside it.  At N > 1 the collective and the
    # combine stay eager on the same stream (every rank issues exactly one allgather per step
    # whether or not its own capture succeeded, so a rank falling back cannot desynchronise them)
    graph, graph_err = None, None
    if not args.no_graph:
        try:
            local_only = True
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=stream, capture_error_mode="thread_local"):
                step()
            graph = cg
            torch.cuda.synchronize(dev)
        except Exception as ex:      # (recorded in the JSON line; the eager step is timed instead)
            graph, graph_err = None, f"{type(ex).__name__}: {ex}"[:300]
            torch.cuda.synchronize(dev)
        local_only = False

    def timed_step(k=None):
        if graph is not None:
            with torch.cuda.stream(stream):
                graph.replay()
            if X is not None:
                exchange()
        else:
            step()
    for _ in range(2):                   # warm replays (every rank: one allgather each)
        timed_step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms_step = time_steps(timed_step, K, stream, dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    status = int(g.status_word().item())
    if status != 0:
        raise SystemExit(f"device status word {status} after the timed steps")
    # per-stage device times: the same step run eagerly with the library's stage events
    ms_eager = time_steps(step, K, stream, dev)
    t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step_max = float(t.item())
    # per-stage device times (mean over steps)
    st_ms = {}
    for a, b, name in [(0, 1, "sort"), (1, 2, "decode"), (2, 3, "dp_local"), (3, 4, "dp_fix"),
                       (4, 5, "dp_cascade"), (5, 6, "traceback"), (6, 7, "compact"), (8, 9, "stats")]:
        st_ms[name] = float(np.mean([ev[k][a].elapsed_time(ev[k][b]) for k in range(K)]))
    st_ms["load"] = float(np.mean([ld[k][0].elapsed_time(ld[k][1]) for k in range(K)]))
    if X is not None:
        st_ms["exchange"] = float(np.mean([xe[k][0].elapsed_time(xe[k][1]) for k in range(K)]))
    diag = g.diagnostics(stream)
    res = g.results()
    m = res["m"]
    hbm_gbs, sm_max, peak_src = peaks()
    value = n_total / (ms_step_max / 1e3)
    if X is not None:
        job = X.results()
        job_offsets, job_totals = job["offsets"], job["totals"]
    else:
        job_offsets, job_totals = res["offsets"], res["totals"]
    m_job = int(job_totals["batches"])

    # dominant kernel roofline: SEG-DP is integer-issue-bound
    dom = max((k for k in st_ms if k != "exchange"), key=st_ms.get)
    if dom in ("dp_local", "dp_fix", "dp_cascade"):
        evals = diag["dp_candidate_evals"]
        per_eval = ncu_summary().get("dp_warp_inst_per_eval", DP_WARP_INST_PER_EVAL)
        achieved = evals * per_eval / (st_ms["dp_local"] / 1e3) / 1e12
        peak = SMS * ISSUE_PER_SM * sm_max * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "k_dp_tiles", "achieved": achieved,
                "peak": peak, "unit": "T warp-instr/s", "frac": achieved / peak,
                "traffic": ncu_traffic("k_dp_tiles"),
                "work": f"{evals} candidate evaluations ({evals / max(n, 1):.1f} per query) x {per_eval:.3f} "
                        f"warp instructions each (ncu inst_executed / evaluations)",
                "peak_source": f"{SMS} SMs x {ISSUE_PER_SM} issue slots/clk x {sm_max:.0f} MHz "
                               f"(guide unit counts; MEASURED_PEAKS sm_max_mhz)"}
    else:
        sh = stage_hbm(st_ms, n, m, diag["sort_passes"], hbm_gbs, diag["sort_key_bits"] != 64)
        key = {"sort": "sort", "decode": "sort", "stats": "stats", "load": "load", "traceback": "traceback",
               "compact": "compact"}.get(dom, "sort")
        roof = {"bound": "hbm", "kernel": dom, "achieved": sh[key]["achieved_gbs"], "peak": hbm_gbs, "unit": "GB/s",
                "frac": sh[key]["frac"], "traffic": ncu_traffic(dom)}
    comp = compulsory_bytes(n_total, m_job)
    step_hbm = {"compulsory_bytes": comp, "achieved_gbs": comp / (ms_step_max / 1e3) / 1e9,
                "peak_gbs": hbm_gbs, "frac": comp / (ms_step_max / 1e3) / 1e9 / hbm_gbs / world,
                "per_gpu": True, "peak_source": peak_src}

    # e2e: the C-ABI with HOST buffers (pinned), H2D/D2H inside the timed region.  The public
    # host-buffer entry point uellm_schedule_pipelined cuts the rank's job into window groups and
    # overlaps group g's compute with the PCIe copies of its neighbours.  N > 1: the ranks' host
    # totals are then combined through the library (one allgather of the 128-byte totals records).
    e2e = None
    if not args.no_e2e:
        import ctypes
        p_in = torch.from_numpy(inp.view(np.int32)).pin_memory()
        p_out = torch.from_numpy(out.view(np.int32)).pin_memory()
        p_slo = torch.from_numpy(slo).pin_memory()
        h_order = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
        h_offs = torch.empty(n + 1, dtype=torch.int32).pin_memory()
        h_nb = np.zeros(1, np.uint64)
        h_tot = U.Totals()
        groups = args.e2e_groups
        pwsb = U.pipeline_workspace_bytes(n, g.cfg, groups)
        pws = torch.empty(pwsb, dtype=torch.uint8, device=dev)
        if world > 1:
            t_rec = torch.zeros(U.TOTALS_BYTES, dtype=torch.uint8).pin_memory()
            d_rec = torch.zeros(U.TOTALS_BYTES, dtype=torch.uint8, device=dev)
            d_all = torch.zeros(world * U.TOTALS_BYTES, dtype=torch.uint8, device=dev)
            h_job = torch.zeros(U.TOTALS_BYTES, dtype=torch.uint8).pin_memory()
            d_job = torch.zeros(U.TOTALS_BYTES, dtype=torch.uint8, device=dev)

        def e2e_step(k=None):
            U.schedule_pipelined(n, p_in, p_out, p_slo, g.cfg, groups, pws, pwsb, h_order, h_offs, h_nb,
                                 ctypes.addressof(h_tot), stream)
            if world > 1:
                ctypes.memmove(t_rec.data_ptr(), ctypes.addressof(h_tot), U.TOTALS_BYTES)
                with torch.cuda.stream(stream):
                    d_rec.copy_(t_rec, non_blocking=True)
                    if args.dist_backend == "nccl":
                        dist.all_gather_into_tensor(d_all, d_rec)
                    else:
                        dist.all_gather(list(d_all.view(world, -1).unbind(0)), d_rec)
                U.totals_combine(d_all, world, U.TOTALS_BYTES, d_job, stream=stream)
                with torch.cuda.stream(stream):
                    h_job.copy_(d_job, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        te = torch.tensor([time_steps(e2e_step, K, stream, dev)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        mh = int(h_nb[0])
        e2e = {"value": n_total / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 12 * n + (U.TOTALS_BYTES if world > 1 else 0),
               "d2h_bytes_per_step": 4 * n + 4 * (mh + 1) + 8 + U.TOTALS_BYTES * (2 if world > 1 else 1),
               "ms_per_step": float(te.item()), "api": f"uellm_schedule_pipelined ({groups or 12} window groups)",
               "exchange": None if world == 1 else "allgather of the ranks' totals records + uellm_totals_combine "
                                                   "(each rank keeps its own order / offsets in host memory)"}
        assert mh == m and h_tot.dp_cost == res["totals"]["dp_cost"], "host-buffer path disagrees with the device path"
        if world > 1:
            jt = U.Totals.from_buffer_copy(h_job.numpy().tobytes())
            assert jt.dp_cost == job_totals["dp_cost"], "e2e job totals disagree with the device exchange"

    # weak-scaling extra (N > 1): every rank schedules the WHOLE job (per-GPU work fixed)
    weak = None
    if world > 1 and not args.no_weak:
        gw = GpuScheduler(n_total, cfg, device=dev, per_batch=False)
        w_in = torch.from_numpy(inp_all.view(np.int32)).to(dev)
        w_out = torch.from_numpy(out_all.view(np.int32)).to(dev)
        w_slo = torch.from_numpy(slo_all).to(dev)

        def wstep(k=None):
            gw.load(w_in, w_out, w_slo, stream)
            gw.schedule(stream)
            gw.stats(stream)
        for _ in range(Wm):
            wstep()
        torch.cuda.synchronize(dev)
        dist.barrier()
        tw = torch.tensor([time_steps(wstep, K, stream, dev)], dtype=torch.float64, device=dev)
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        weak = {"scaling": "weak", "queries_per_rank": n_total, "ms_per_step": float(tw.item()),
                "value": world * n_total / (float(tw.item()) / 1e3), "unit": UNIT}
        del gw, w_in, w_out, w_slo
        torch.cuda.empty_cache()

    next_rows = {}
    if world == 1 and not args.no_sim:
        next_rows = run_next_rows(args, g, cfg, n, d_in, d_out, d_slo, m, stream, dev, hbm_gbs, K, Wm)

    configs = {}
    if world == 1 and not args.no_configs and args.n is None and args.config == "c4":
        for name in ("c2", "c3", "c5"):
            configs[name] = sub_config(name, K, Wm, stream, dev, hbm_gbs)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        cpu = cpu_baseline(inp, out, slo, cfg, windows=min(cores, max(1, n // (cfg.window or n))))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm,
            "ms_per_step": ms_step_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (workloads seeded generator; one job, seed 0)",
            "config": {"workload": desc, "queries": n_total, "queries_rank0": n, "window": cfg.window,
                       "max_batch": cfg.max_batch, "lambda_us": cfg.lambda_us,
                       "l2": "inputs 1.2 GB >> 126 MB L2; no flush needed",
                       "parallelism": f"{world} rank(s), contiguous window blocks of one job; a9: one allgather "
                                      f"of [totals | boundary bitmap] records, job rebuilt on every rank"},
            "step_launch": {"cuda_graph": graph is not None, "graph_error": graph_err,
                            "eager_ms_per_step": ms_eager,
                            "load": "uellm_profile_reload (device-side validation, no host sync); "
                                    "one synchronising uellm_profile_load before the timed region"},
            "roofline": roof, "step_hbm_roofline": step_hbm,
            "stage_hbm": stage_hbm(st_ms, n, m, diag["sort_passes"], hbm_gbs, diag["sort_key_bits"] != 64),
            "stage_ms": st_ms,
            # our kernels launched inside the timed region: K steps x (reload [load / fused pack +
            # status check] + schedule + stats [+ a9])
            "gpu_launches": K * int(diag["sched_launches"] + diag["stats_launches"] + 2 + (4 if world > 1 else 0)),
            "gpu_launches_per_step": int(diag["sched_launches"] + diag["stats_launches"] + 2 + (4 if world > 1 else 0)),
            "diagnostics": diag, "batches": m_job, "dp_cost": job_totals["dp_cost"],
            "job_offsets_sha256": offsets_digest(job_offsets, job_totals),
            "a9_exchange_bytes_per_rank": X.rec_bytes if X else None,
            "weak_scaling": weak, "configs": configs,
            "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "next_rows": next_rows,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_next_rows(args, g, cfg, n, d_in, d_out, d_slo, m, stream, dev, hbm_gbs, K, Wm):
    """NEXT rows on the same resident stream, each timed on its own (N = 1)."""
    import torch
    import workloads as W
    from paper_2409_14961_b200 import uellm as U
    from paper_2409_14961_b200.scheduler import GpuScheduler
    rank = 0
    next_rows = {}
    # f2: the sequential-execution simulator over this step's schedule (Poisson arrivals resident
    # in HBM, per-batch ends and per-query latencies written)
    arr = W.poisson_arrivals(n, rank, W.MEAN_GAP_US.get(args.config, 21_000))
    d_arr = torch.from_numpy(arr.view(np.int64)).to(dev)
    for _ in range(max(Wm, 1)):
        g.simulate(d_arr, stream)
    sim_ms = time_steps(lambda k: g.simulate(d_arr, stream), K, stream, dev)
    sim = g.sim_results()["totals"]
    alg_b = 32 * n + 12 * m          # arrival 8 + order/in/out/slo 4 each + latency 8 per query; offsets 4 + end 8 per batch
    next_rows["f2_simulate"] = {
        "ms": sim_ms, "queries_per_s": n / (sim_ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": alg_b / (sim_ms / 1e3) / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": alg_b / (sim_ms / 1e3) / 1e9 / hbm_gbs, "algorithmic_bytes": alg_b},
        "arrivals": f"Poisson, mean gap {W.MEAN_GAP_US.get(args.config, 21_000)} us",
        "totals": {k: sim[k] for k in ("makespan_us", "idle_us", "viol", "mean_latency_s",
                                        "slo_violation_rate", "utilization", "throughput_tok_s")}}

    # f4: profiler stand-ins + monitor producing the predicted lengths of a stream of this size
    tl = torch.from_numpy(W.true_output_lengths(n, rank).view(np.int32)).to(dev)
    pr = torch.empty(n, dtype=torch.int32, device=dev)
    st0 = U.MonitorState()
    st0.inflation_factor = 1.0
    init = torch.frombuffer(bytearray(bytes(st0)), dtype=torch.uint8).to(dev)
    state = init.clone()
    pc = W.PredictorConfig(variant=2, error_rate=0.0049, bucket_width=16, window=cfg.window or n, seed=rank)
    cp = U.make_predictor(pc)
    pwsb = U.predict_workspace_bytes(n, cp)
    pws = torch.empty(max(pwsb, 1), dtype=torch.uint8, device=dev)

    def f4_step(level_ws):
        with torch.cuda.stream(stream):
            state.copy_(init)
        U.predict_lengths(n, tl, cp, state, pr, None, stream, ws=pws if level_ws else None,
                          ws_bytes=pwsb if level_ws else 0)

    f4_ms = {}
    for path, lw in (("window", False), ("level", bool(pwsb))):
        if path == "level" and not lw:
            continue
        for _ in range(max(Wm, 1)):
            f4_step(lw)
        f4_ms[path] = time_steps(lambda k: f4_step(lw), K, stream, dev)
    best = min(f4_ms, key=f4_ms.get)
    pms = f4_ms[best]
    fin = U.MonitorState.from_buffer_copy(state.cpu().numpy().tobytes())
    next_rows["f4_predict"] = {
        "ms": pms, "queries_per_s": n / (pms / 1e3),
        "roofline": {"bound": "hbm", "achieved": 8 * n / (pms / 1e3) / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": 8 * n / (pms / 1e3) / 1e9 / hbm_gbs, "algorithmic_bytes": 8 * n},
        "predictor": "noisy, error 0.0049, 16-token buckets, monitor gamma 1.1 cap 2.0, epoch = window",
        "path": best, "ms_by_path": f4_ms,
        "launches": 4 if best == "level" else (n + (cfg.window or n) - 1) // (cfg.window or n),
        "final_state": {"corrections": fin.corrections, "inflation_factor": fin.inflation_factor}}

    # f1: the paper's own Alg. 1 (SLO-ODBS, parallel greedy) on the same resident stream
    if args.mode == "seg_dp":
        c1 = cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.02, threshold=900.0)
        g1 = GpuScheduler(n, c1, device=dev, per_batch=False)

        def f1_step(k=None):
            g1.load(d_in, d_out, d_slo, stream)
            g1.schedule(stream)
            g1.stats(stream)
        for _ in range(max(Wm, 1)):
            f1_step()
        f1_ms = time_steps(f1_step, K, stream, dev)
        r1 = g1.results()
        nk = ncu_summary().get("next_kernels", {})
        a1 = nk.get("k_alg1_next")
        f1_roof = None
        if a1:
            peak = SMS * ISSUE_PER_SM * peaks()[1] * 1e6 / 1e12
            ach = a1["inst_executed"] / (a1["duration_ms"] / 1e3) / 1e12
            f1_roof = {"bound": "alu", "kernel": "k_alg1_next (one thread per position simulates Alg. 1 from a "
                                                  "fresh batch: FP64 expression trees)",
                       "achieved": ach, "peak": peak, "unit": "T warp-instr/s", "frac": ach / peak,
                       "source": "ncu inst_executed / duration of the kernel (profiles/ncu_summary.json next_kernels)",
                       "share_of_f1_ms": a1["duration_ms"] / f1_ms}
        next_rows["f1_slo_odbs"] = {
            "ms": f1_ms, "queries_per_s": n / (f1_ms / 1e3), "roofline": f1_roof,
            "algorithm": "Alg. 1 literal (w1=1, w2=0.02, threshold=900), load + schedule + stats",
            "batches": r1["m"], "dp_objective_of_its_schedule": r1["totals"]["dp_cost"]}
        del g1
        torch.cuda.empty_cache()

    # f3: HELR deployer on a 20-device B200 topology (3 nodes of 8, truncated to the 20-device
    # limit; LLaMA-2-70B fp16, 80 layers): 2^20 x 20 DP states, 20 popcount levels
    t = W.b200_cluster(nodes=3, per_node=8, seed=rank)
    t = t.replace(memory_bytes=t.memory_bytes[:20], performance=t.performance[:20],
                  link_latency_s=np.ascontiguousarray(t.link_latency_s[:20, :20]))
    hb = U.helr_workspace_bytes(20)
    hws = torch.empty(hb, dtype=torch.uint8, device=dev)
    hout = torch.zeros(U.C.sizeof(U.DeviceMap), dtype=torch.uint8, device=dev)
    for _ in range(max(Wm, 1)):
        U.helr_plan(t, hws, hb, hout, stream)
    hms = time_steps(lambda k: U.helr_plan(t, hws, hb, hout, stream), K, stream, dev)
    dm = U.DeviceMap.from_buffer_copy(hout.cpu().numpy().tobytes()).as_dict()
    bg = U.bgs_plan(t, hws, hb).as_dict()           # the paper's baseline deployer, for context
    import math
    relax = sum(math.comb(20, k) * k * (k - 1) for k in range(1, 21))
    next_rows["f3_helr"] = {
        "ms": hms, "devices": 20, "dp_states": (1 << 20) * 20, "relaxations": relax,
        "relaxations_per_s": relax / (hms / 1e3),
        # compulsory traffic: every DP entry (8 B value + 1 B argument) written once and read back
        # by its successors at the next level at least once
        "roofline": {"bound": "latency", "note": "20 dependent popcount levels, one launch each; the DP "
                     "table (2^20 x 20 x 9 B) is written once and read once at least",
                     "dram_table_bytes": (1 << 20) * 20 * 9,
                     "achieved_gbs": 2 * (1 << 20) * 20 * 9 / (hms / 1e3) / 1e9, "peak_gbs": hbm_gbs,
                     "frac": 2 * (1 << 20) * 20 * 9 / (hms / 1e3) / 1e9 / hbm_gbs},
        "device_map": {"devices": dm["devices"], "layer_count": dm["layer_count"],
                       "latency_s": dm["latency_s"], "objective": dm["objective"]},
        "bgs_baseline": {"devices": bg["devices"], "latency_s": bg["latency_s"], "objective": bg["objective"]}}
    return next_rows


if __name__ == "__main__":
    main()
