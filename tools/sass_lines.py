#!/usr/bin/env python
"""Per-source-line instruction counts of one kernel: joins the SASS page of an ncu report
(`ncu -i REP --page source --csv -k KERNEL`, per-address "Instructions Executed" and stall samples)
with the line table of the same build (`nvdisasm -gi` of the cubin in the object file).

  python tools/sass_lines.py OBJ.o KERNEL_MANGLED NCU_SOURCE.csv [SRC_FILE_SUBSTR]

Prints the source lines of SRC_FILE_SUBSTR (default k_segdp.cu) by share of executed warp
instructions, plus an opcode histogram (the committed SASS evidence of profiles/)."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel, src):
    d = tempfile.mkdtemp()
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d,
                          stdout=subprocess.DEVNULL)
    cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.check_output(["nvdisasm", "-gi", os.path.join(d, cubin)], text=True)
    lines, ops = {}, {}
    cur = None
    inside = False
    in_chain = False             # consecutive '//##' comments: innermost first, then its callers
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + kernel
            cur = None
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            f, l = m.group(1), int(m.group(2))
            if in_chain and cur is not None:
                continue
            in_chain = True
            if src in f:
                cur = l                   # innermost location in the source file
            else:
                mm = re.search(r'inlined at "([^"]+)", line (\d+)', ln)
                if mm and src in mm.group(1):
                    cur = int(mm.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        in_chain = False
        if m:
            a = int(m.group(1), 16)
            lines[a] = cur
            ops[a] = m.group(3).split(".")[0]
    return lines, ops


def main():
    obj, kernel, csvp = sys.argv[1:4]
    src = sys.argv[4] if len(sys.argv) > 4 else "k_segdp.cu"
    lines, ops = line_table(obj, kernel, src)
    rows = list(csv.reader(open(csvp)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    i0 = rows.index(hdr)
    ia = hdr.index("Address")
    ie = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    by_line = collections.Counter()
    samp_line = collections.Counter()
    by_op = collections.Counter()
    tot = 0
    tots = 0
    base = None
    isrc = hdr.index("Source")
    for r in rows[i0 + 1:]:
        if len(r) <= ie or not r[ia].startswith("0x"):
            continue
        if base is None:
            base = int(r[ia], 16)        # ncu prints load addresses: rebase to the function start
        a = int(r[ia], 16) - base
        ops[a] = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0].split(".")[0]
        n = float(r[ie] or 0)
        s = float(r[isamp] or 0)
        tot += n
        tots += s
        by_line[lines.get(a)] += n
        samp_line[lines.get(a)] += s
        by_op[ops.get(a, "?")] += n
    print(f"# {kernel}: {tot:.4g} warp instructions executed, {tots:.0f} stall samples")
    print("line,warp_inst,share_pct,samples_share_pct")
    for l, n in by_line.most_common(60):
        print(f"{l},{n:.0f},{100 * n / tot:.2f},{100 * samp_line[l] / max(tots, 1):.2f}")
    print("\nopcode,warp_inst,share_pct")
    for o, n in by_op.most_common(40):
        print(f"{o},{n:.0f},{100 * n / tot:.2f}")


if __name__ == "__main__":
    main()
