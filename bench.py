#!/usr/bin/env python
"""Benchmark of the UELLM batch-scheduler hot path on B200 (BASELINE.json metric:
"queries scheduled/sec (device-timed, max over ranks) and HBM GB/s vs roofline").

One step = one pass of the whole hot path over one batch of synthetic queries resident in HBM:
uellm_profile_load (validate + SLO->us + key pack) -> uellm_schedule_batches (radix sort,
SEG-DP, traceback, offsets) -> uellm_batch_stats (per-batch stats + totals), plus, at N > 1,
the allgather of per-rank totals (a9).  Workload at N = 1: BJ configs[3] (10^8 queries in
10^6-query windows, c4).  Weak scaling: every rank schedules its own 10^8-query stream.

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
    k = ncu_summary().get("kernels", {}).get(kernel)
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
    nq = nwin * wl
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
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": desc, "sample_queries": nq, "windows": nwin},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, nwin), "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{nwin} windows x {wl} queries per step, one window per thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--no-sim", action="store_true", help="skip the NEXT-row timings (f2, f3, f4)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo only for multi-rank tests on one GPU)")
    ap.add_argument("--e2e-groups", type=int, default=0, help="window groups of the pipelined e2e call (0 = 12)")
    ap.add_argument("--dp-tile", type=int, default=0, help="SEG-DP tile length override (tuning only)")
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
    from paper_2409_14961_b200.distributed import GATHER_WORDS, combine_totals
    from paper_2409_14961_b200.scheduler import GpuScheduler

    local = local % max(torch.cuda.device_count(), 1)   # (test runs may put several ranks on one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    def allgather(out_buf, in_buf):
        """a9: one collective; NCCL's allgather into one tensor (gloo, for tests: list form)."""
        if args.dist_backend == "nccl":
            dist.all_gather_into_tensor(out_buf, in_buf)
        else:
            dist.all_gather(list(out_buf.view(world, -1).unbind(0)), in_buf)
    desc, inp, out, slo, cfg = workload(args.config, rank, args.n)
    if args.dp_tile:
        cfg = cfg.replace(dp_tile=args.dp_tile)
    if args.mode != "seg_dp":
        import workloads as W
        cfg = cfg.replace(mode={"slo_odbs": W.MODE_SLO_ODBS, "fifo": W.MODE_FIFO, "sort_only": W.MODE_SORT_ONLY}[args.mode],
                          w1=1.0, w2=0.02, threshold=900.0)
        desc += f"; mode {args.mode} (Alg. 1: w1=1, w2=0.02, threshold=900)" if args.mode == "slo_odbs" else f"; mode {args.mode}"
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
    with torch.cuda.stream(stream):
        for row in ev:
            for e in row:
                e.record(stream)          # materialise the cudaEvent_t handles
    # a9 exchange buffer: [16 totals words | boundary bitmap of this rank's positions] (every rank
    # schedules n queries, so the buffers have one size)
    xw = D.exchange_words(n)
    gather_buf = torch.zeros(world * xw, dtype=torch.int64, device=dev)
    gather_in = torch.zeros(xw, dtype=torch.int64, device=dev)
    bm_view = D.bitmap_view(gather_in)

    def step(k=None):
        if k is not None:
            ld[k][0].record(stream)
        g.load(d_in, d_out, d_slo, stream)
        if k is not None:
            ld[k][1].record(stream)
            U.set_stage_events(g.profile, ev[k])
        g.schedule(stream)
        g.stats(stream)
        if world > 1:   # a9: ONE NCCL allgather of per-rank totals + batch-boundary bitmap
            U.boundary_bitmap(g.profile, g.cfg, bm_view, stream)
            with torch.cuda.stream(stream):
                gather_in[:13].copy_(g.totals.view(torch.int64)[:13])
                allgather(gather_buf, gather_in)

    for _ in range(Wm):
        step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(K):
        step(k)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_total = t0.elapsed_time(t1)
    ms_step = ms_total / K
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
    diag = g.diagnostics(stream)
    res = g.results()
    m = res["m"]
    hbm_gbs, sm_max, peak_src = peaks()
    value = world * n / (ms_step_max / 1e3)

    # dominant kernel roofline
    dom = max(st_ms, key=st_ms.get)
    if dom in ("dp_local", "dp_fix", "dp_cascade"):
        # SEG-DP is integer-issue-bound: units = candidate evaluations counted live by the kernel,
        # per-unit cost = warp instructions per evaluation from the committed ncu capture
        # (profiles/ncu_summary.json); peak = 148 SMs x 4 schedulers x 1 warp-instr/clk x max clock
        evals = diag["dp_candidate_evals"]
        per_eval = ncu_summary().get("dp_warp_inst_per_eval", DP_WARP_INST_PER_EVAL)
        achieved = evals * per_eval / (st_ms["dp_local"] / 1e3) / 1e12
        peak = SMS * ISSUE_PER_SM * sm_max * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "k_dp_tiles", "achieved": achieved,
                "peak": peak, "unit": "T warp-instr/s", "frac": achieved / peak,
                "traffic": ncu_traffic("k_dp_tiles"),
                "work": f"{evals} candidate evaluations ({evals / n:.1f} per query) x {per_eval:.3f} "
                        f"warp instructions each (ncu inst_executed / evaluations)",
                "peak_source": f"{SMS} SMs x {ISSUE_PER_SM} issue slots/clk x {sm_max:.0f} MHz "
                               f"(guide unit counts; MEASURED_PEAKS sm_max_mhz)"}
    else:
        # HBM-bound stages: algorithmic bytes per launch of the stage
        alg = {"sort": 24 * n * diag["sort_passes"], "decode": 24 * n, "stats": 12 * n + 80 * m,
               "load": 24 * n, "traceback": 2 * n, "compact": n // 8 + 4 * m}.get(dom, 0)
        achieved = alg / (st_ms[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                "frac": achieved / hbm_gbs, "traffic": ncu_traffic(dom)}
    comp = compulsory_bytes(n, m)
    step_hbm = {"compulsory_bytes": comp, "achieved_gbs": comp / (ms_step_max / 1e3) / 1e9,
                "peak_gbs": hbm_gbs, "frac": comp / (ms_step_max / 1e3) / 1e9 / hbm_gbs,
                "peak_source": peak_src}

    # e2e: the C-ABI with HOST buffers (pinned), H2D/D2H inside the timed region.  The public
    # host-buffer entry point uellm_schedule_pipelined cuts the job into window groups and overlaps
    # group g's compute with the PCIe copies of its neighbours (same results as the three calls).
    e2e = None
    if not args.no_e2e:
        import ctypes
        p_in = torch.from_numpy(inp.view(np.int32)).pin_memory()
        p_out = torch.from_numpy(out.view(np.int32)).pin_memory()
        p_slo = torch.from_numpy(slo).pin_memory()
        h_order = torch.empty(n, dtype=torch.int32).pin_memory()
        h_offs = torch.empty(n + 1, dtype=torch.int32).pin_memory()
        h_nb = np.zeros(1, np.uint64)
        h_tot = U.Totals()
        groups = args.e2e_groups
        pwsb = U.pipeline_workspace_bytes(n, g.cfg, groups)
        pws = torch.empty(pwsb, dtype=torch.uint8, device=dev)

        def e2e_step():
            U.schedule_pipelined(n, p_in, p_out, p_slo, g.cfg, groups, pws, pwsb, h_order, h_offs, h_nb,
                                 ctypes.addressof(h_tot), stream)
            if world > 1:
                with torch.cuda.stream(stream):
                    gather_in[:13].copy_(torch.from_numpy(np.frombuffer(bytes(h_tot), np.int64)[:13].copy()),
                                         non_blocking=False)
                    allgather(gather_buf, gather_in)
        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        te = torch.tensor([e0.elapsed_time(e1) / K], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        mh = int(h_nb[0])
        e2e = {"value": world * n / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 12 * n, "d2h_bytes_per_step": 4 * n + 4 * (mh + 1) + 8 + U.TOTALS_BYTES,
               "ms_per_step": float(te.item()), "api": f"uellm_schedule_pipelined ({groups or 12} window groups)",
               "exchange": "N > 1: allgather of the per-rank totals (the boundaries are already in each rank's host buffers)"}
        assert mh == m and h_tot.dp_cost == res["totals"]["dp_cost"], "host-buffer path disagrees with the device path"

    # NEXT f2: the sequential-execution simulator over this step's schedule, timed on its own
    # (not part of the a1-a9 step): Poisson arrivals resident in HBM, per-batch ends and
    # per-query latencies written
    next_rows = {}
    if not args.no_sim:
        import workloads as W
        arr = W.poisson_arrivals(n, rank, W.MEAN_GAP_US.get(args.config, 21_000))
        d_arr = torch.from_numpy(arr.view(np.int64)).to(dev)
        for _ in range(max(Wm, 1)):
            g.simulate(d_arr, stream)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(K):
            g.simulate(d_arr, stream)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        sim_ms = s0.elapsed_time(s1) / K
        sim = g.sim_results()["totals"]
        alg_b = 32 * n + 12 * m          # arrival 8 + order/in/out/slo 4 each + latency 8 per query; offsets 4 + end 8 per batch
        next_rows["f2_simulate"] = {
            "ms": sim_ms, "queries_per_s": n / (sim_ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": alg_b / (sim_ms / 1e3) / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                         "frac": alg_b / (sim_ms / 1e3) / 1e9 / hbm_gbs, "algorithmic_bytes": alg_b},
            "arrivals": f"Poisson, mean gap {W.MEAN_GAP_US.get(args.config, 21_000)} us",
            "totals": {k: sim[k] for k in ("makespan_us", "idle_us", "viol", "mean_latency_s",
                                            "slo_violation_rate", "utilization", "throughput_tok_s")}}

    # NEXT f4: profiler stand-ins + monitor producing the predicted lengths of a stream of this
    # step's size (true lengths resident in HBM; one monitor epoch per scheduling window)
    if not args.no_sim:
        import workloads as W
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
            p0 = torch.cuda.Event(enable_timing=True)
            p1 = torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            for _ in range(K):
                f4_step(lw)
            p1.record(stream)
            torch.cuda.synchronize(dev)
            f4_ms[path] = p0.elapsed_time(p1) / K
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

    # NEXT f1: the paper's own Alg. 1 (SLO-ODBS, parallel greedy) on the same resident stream
    if not args.no_sim and args.mode == "seg_dp":
        import workloads as W
        c1 = cfg.replace(mode=W.MODE_SLO_ODBS, w1=1.0, w2=0.02, threshold=900.0)
        g1 = GpuScheduler(n, c1, device=dev, per_batch=False)

        def f1_step():
            g1.load(d_in, d_out, d_slo, stream)
            g1.schedule(stream)
            g1.stats(stream)
        for _ in range(max(Wm, 1)):
            f1_step()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(K):
            f1_step()
        a1.record(stream)
        torch.cuda.synchronize(dev)
        f1_ms = a0.elapsed_time(a1) / K
        r1 = g1.results()
        next_rows["f1_slo_odbs"] = {
            "ms": f1_ms, "queries_per_s": n / (f1_ms / 1e3),
            "algorithm": "Alg. 1 literal (w1=1, w2=0.02, threshold=900), load + schedule + stats",
            "batches": r1["m"], "dp_objective_of_its_schedule": r1["totals"]["dp_cost"]}
        del g1
        torch.cuda.empty_cache()

    # NEXT f3: HELR deployer on a 20-device B200 topology (3 nodes of 8, truncated to the 20-device
    # limit; LLaMA-2-70B fp16, 80 layers): 2^20 x 20 DP states, 20 popcount levels
    if not args.no_sim:
        import workloads as W
        t = W.b200_cluster(nodes=3, per_node=8, seed=rank)
        t = t.replace(memory_bytes=t.memory_bytes[:20], performance=t.performance[:20],
                      link_latency_s=np.ascontiguousarray(t.link_latency_s[:20, :20]))
        hb = U.helr_workspace_bytes(20)
        hws = torch.empty(hb, dtype=torch.uint8, device=dev)
        hout = torch.zeros(U.C.sizeof(U.DeviceMap), dtype=torch.uint8, device=dev)
        for _ in range(max(Wm, 1)):
            U.helr_plan(t, hws, hb, hout, stream)
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(K):
            U.helr_plan(t, hws, hb, hout, stream)
        h1.record(stream)
        torch.cuda.synchronize(dev)
        hms = h0.elapsed_time(h1) / K
        dm = U.DeviceMap.from_buffer_copy(hout.cpu().numpy().tobytes()).as_dict()
        bg = U.bgs_plan(t, hws, hb).as_dict()           # the paper's baseline deployer, for context
        import math
        relax = sum(math.comb(20, k) * k * (k - 1) for k in range(1, 21))
        next_rows["f3_helr"] = {
            "ms": hms, "devices": 20, "dp_states": (1 << 20) * 20, "relaxations": relax,
            "relaxations_per_s": relax / (hms / 1e3),
            "roofline": {"bound": "latency", "note": "20 dependent popcount levels; the DP table "
                         "(168 MB) streams once per level", "dram_table_bytes": (1 << 20) * 20 * 9},
            "device_map": {"devices": dm["devices"], "layer_count": dm["layer_count"],
                           "latency_s": dm["latency_s"], "objective": dm["objective"]},
            "bgs_baseline": {"devices": bg["devices"], "latency_s": bg["latency_s"], "objective": bg["objective"]}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        cpu = cpu_baseline(inp, out, slo, cfg, windows=min(cores, max(1, n // (cfg.window or n))))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm,
            "ms_per_step": ms_step_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (workloads.c4 seeded generator, rank = seed)",
            "config": {"workload": desc, "queries_per_rank": n, "window": cfg.window,
                       "max_batch": cfg.max_batch, "lambda_us": cfg.lambda_us,
                       "l2": "inputs 1.2 GB/rank >> 126 MB L2; no flush needed",
                       "parallelism": f"{world} rank(s), windows independent, one allgather of totals + boundary bitmaps"},
            "roofline": roof, "step_hbm_roofline": step_hbm, "stage_ms": st_ms,
            # our kernels launched inside the timed region: K steps x (load + schedule + stats)
            "gpu_launches": K * int(diag["sched_launches"] + diag["stats_launches"] + 1),
            "gpu_launches_per_step": int(diag["sched_launches"] + diag["stats_launches"] + 1),
            "diagnostics": diag, "batches": m, "dp_cost": res["totals"]["dp_cost"],
            "job_totals": ({k: v for k, v in combine_totals(gather_buf.view(world, xw)[:, :GATHER_WORDS]).items()
                            if k in ("n", "batches", "dp_cost", "viol_alone")} if world > 1 else None),
            "a9_exchange_bytes_per_rank": 8 * xw,
            "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "next_rows": next_rows,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
