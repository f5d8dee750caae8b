#!/usr/bin/env python
"""Summarise an ncu capture + launch list into profiles/ (committed evidence).

  python profiles/summarize.py --rep gpurun_out/prof_full_r01c.ncu-rep \
      --launches gpurun_out/launches_r01c.csv --bench gpurun_out/bench_r01c.json --tag r01

Writes profiles/<tag>_launch_shares.csv, profiles/<tag>_ncu_summary.md and
profiles/ncu_summary.json (read by bench.py for the roofline `traffic` field and the SEG-DP
warp-instructions-per-evaluation figure)."""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))


def kname(s):
    return s.split("(")[0].replace("void ", "").replace("uellm::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", default=None, help=".ncu-rep (or pass --raw)")
    ap.add_argument("--raw", default=None, help="csv of `ncu -i REP --page raw --csv`")
    ap.add_argument("--launches", required=True)
    ap.add_argument("--bench", required=True)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--steps", type=int, default=2, help="c4 steps in the launch list")
    ap.add_argument("--next-raw", default=None, help="raw csv of an ncu capture of the NEXT-row kernels")
    a = ap.parse_args()
    bench = json.loads(open(a.bench).read().strip().splitlines()[-1])
    evals = bench["diagnostics"]["dp_candidate_evals"]
    steps_in_launch_list = a.steps

    # launch shares
    rows = list(csv.reader(open(a.launches)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    data = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]
    agg, cnt = defaultdict(float), defaultdict(int)
    for d in data:
        if d.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
            continue
        agg[kname(d["Kernel Name"])] += float(d["Metric Value"])
        cnt[kname(d["Kernel Name"])] += 1
    tot = sum(agg.values())
    lines = [f"# {a.tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none) of "
             "`bench.py --steps 1 --warmup 1 --no-configs` (c4 steps + NEXT rows); cold-cache, serialised: "
             "compare shares, not absolutes",
             "kernel,launches,total_ns,share_pct"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{k},{cnt[k]},{v:.0f},{100 * v / tot:.2f}")
    open(os.path.join(HERE, f"{a.tag}_launch_shares.csv"), "w").write("\n".join(lines) + "\n")

    # full capture
    raw = (open(a.raw).read() if a.raw else
           subprocess.check_output(["ncu", "-i", a.rep, "--page", "raw", "--csv"]).decode())
    rr = list(csv.reader(io.StringIO(raw)))
    h, units, body = rr[0], rr[1], rr[2:]
    ix = {n: h.index(n) for n in h}

    def val(r, n, scale=1.0):
        u = units[ix[n]]
        f = float(r[ix[n]])
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(u, 1.0)
        return f * mult * scale

    K, seen = {}, defaultdict(int)
    for r in body:
        n = kname(r[ix["Kernel Name"]])
        key = n if not seen[n] else f"{n}#{seen[n]}"
        seen[n] += 1
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        dur = val(r, "gpu__time_duration.sum")
        K[key] = {"duration_ms": dur, "dram_read_bytes": rd, "dram_write_bytes": wr,
                  "dram_bytes_per_launch": rd + wr, "dram_gbs": (rd + wr) / dur / 1e6,
                  "inst_executed": float(r[ix["smsp__inst_executed.sum"]]),
                  "l2_bytes": float(r[ix["lts__t_sectors.sum"]]) * 32.0,
                  "issue_active_pct": float(r[ix["smsp__issue_active.avg.pct_of_peak_sustained_active"]]),
                  "warps_active_pct": float(r[ix["sm__warps_active.avg.pct_of_peak_sustained_active"]]),
                  "registers": int(float(r[ix["launch__registers_per_thread"]]))}
    dp = next(v for k, v in K.items() if k.startswith("k_dp_tiles"))
    summ = {"round": a.tag, "source": f"ncu --set full --clock-control none; {os.path.basename(a.rep or a.raw)}; "
                                     "bench.py c4 (1e8 queries, seed 0), one step",
            "dp_candidate_evals_c4_seed0": evals,
            "dp_warp_inst_per_eval": dp["inst_executed"] / evals, "kernels": K}
    if a.next_raw:
        nr = list(csv.reader(open(a.next_raw)))
        nh, nu, nb = nr[0], nr[1], nr[2:]
        nix = {n_: nh.index(n_) for n_ in nh}
        NK = {}
        for r in nb:
            nm = kname(r[nix["Kernel Name"]]).split("<")[0]
            if nm in NK:
                continue                       # first launch of each kernel
            u = nu[nix["gpu__time_duration.sum"]]
            dur = float(r[nix["gpu__time_duration.sum"]]) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(u, 1.0)
            NK[nm] = {"duration_ms": dur, "inst_executed": float(r[nix["smsp__inst_executed.sum"]]),
                      "issue_active_pct": float(r[nix["smsp__issue_active.avg.pct_of_peak_sustained_active"]]),
                      "dram_bytes_per_launch": float(r[nix["dram__bytes_read.sum"]]) + float(r[nix["dram__bytes_write.sum"]])}
        summ["next_kernels"] = NK
    json.dump(summ, open(os.path.join(HERE, "ncu_summary.json"), "w"), indent=1)
    md = [f"# {a.tag} ncu summary (B200, c4 = 10^8 queries, one step)", "",
          f"Bench line of the same code: {bench['value']:.3e} q/s, {bench['ms_per_step']:.2f} ms/step "
          f"(stage ms: " + ", ".join(f"{k} {v:.2f}" for k, v in bench["stage_ms"].items()) + ").", "",
          "| kernel | ms (ncu) | DRAM read GB | DRAM write GB | DRAM GB/s | L2 GB/s | issue active % | warps active % | regs |",
          "|---|---|---|---|---|---|---|---|---|"]
    for k, v in K.items():
        md.append(f"| {k} | {v['duration_ms']:.3f} | {v['dram_read_bytes'] / 1e9:.3f} | "
                  f"{v['dram_write_bytes'] / 1e9:.3f} | {v['dram_gbs']:.0f} | {v['l2_bytes'] / v['duration_ms'] / 1e6:.0f} | "
                  f"{v['issue_active_pct']:.1f} | "
                  f"{v['warps_active_pct']:.1f} | {v['registers']} |")
    md += ["", f"SEG-DP: {dp['inst_executed'] / 1e8:.1f} warp instructions per query, "
               f"{summ['dp_warp_inst_per_eval']:.3f} per candidate evaluation ({evals / 1e8:.1f} evaluations per query)."]
    open(os.path.join(HERE, f"{a.tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
