#!/usr/bin/env python
"""Summary of an ncu SASS source page (`ncu -i REP --page source --csv -k KERNEL`): total executed warp
instructions, stall-reason shares of the warp samples, opcode histogram and the hottest instructions.
usage: python tools/ncu_sass_summary.py SOURCE.csv [TOP]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    ix = {h: i for i, h in enumerate(hdr)}
    inst = [int(r[ix["Instructions Executed"]] or 0) for r in body]
    samp = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body]
    tot_i, tot_s = sum(inst), sum(samp)
    print(f"{rows[0][1][:90]}\nwarp instructions {tot_i:.4g}, samples {tot_s}")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(int(r[ix[h]] or 0) for r in body) for h in stalls}
    print("stalls:", ", ".join(f"{h[6:]} {100 * v / max(tot_s, 1):.1f}%" for h, v in
                                sorted(agg.items(), key=lambda x: -x[1]) if v))
    ops = collections.Counter()
    for r, n in zip(body, inst):
        op = r[ix["Source"]].split()
        op = [o for o in op if not o.startswith("@")]
        if op:
            ops[op[0].split(".")[0]] += n
    print("opcodes:", ", ".join(f"{k} {100 * v / max(tot_i, 1):.1f}%" for k, v in ops.most_common(14)))
    order = sorted(range(len(body)), key=lambda k: -samp[k])[:top]
    for k in order:
        r = body[k]
        print(f"{r[ix['Address']][-5:]} {inst[k]:>11} {100 * samp[k] / max(tot_s, 1):5.1f}%  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main()
