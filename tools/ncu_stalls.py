#!/usr/bin/env python3
"""Aggregate ncu source-page (SASS) stall samples per kernel.

  ncu_stalls.py <report.ncu-rep> [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in txt.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line.split(",", 1)[1].strip().strip(",").strip('"'), []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in blocks:
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    si = h.index("Source")
    ns = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = Counter()
    per = []
    opc = Counter()
    for r in rows[1:]:
        if len(r) <= ns:
            continue
        s = int(r[ns] or 0)
        per.append((s, r[si].strip()))
        op = r[si].strip().split()[0] if r[si].strip() else "?"
        if op.startswith("@"):
            op = r[si].strip().split()[1]
        opc[op.split(".")[0]] += s
        for i in stall_cols:
            tot[h[i]] += int(r[i] or 0)
    # dynamic instruction mix (warp-level instructions executed per opcode)
    ie = next((i for i, c in enumerate(h) if c.strip() == "Instructions Executed"), None)
    mix = Counter()
    if ie is not None:
        for r in rows[1:]:
            if len(r) <= ie or not r[si].strip():
                continue
            op = r[si].strip().split()[0]
            if op.startswith("@"):
                op = r[si].strip().split()[1]
            try:
                mix[op.split(".")[0]] += int(float(r[ie] or 0))
            except ValueError:
                pass
    S = sum(tot.values()) or 1
    print(f"== {name[:90]}  samples {S}")
    if mix:
        M = sum(mix.values()) or 1
        print(f"  executed (warp instructions {M}):", ", ".join(f"{k} {100 * v / M:.1f}%" for k, v in mix.most_common(14)))
    print("  stalls:", ", ".join(f"{k[6:]} {100 * v / S:.1f}%" for k, v in tot.most_common(8)))
    print("  by opcode:", ", ".join(f"{k} {100 * v / S:.1f}%" for k, v in opc.most_common(10)))
    for s, src in sorted(per, reverse=True)[:top]:
        print(f"   {100 * s / S:5.1f}%  {src[:100]}")
