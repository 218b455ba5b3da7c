#!/usr/bin/env python3
"""Summarise ncu outputs into the committed profiles/ text files.

  summarize_ncu.py launches <launches.csv>            per-kernel launch list + shares
  summarize_ncu.py full <report.ncu-rep>              key metrics per profiled launch
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    k, v, mname = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    grid, blk = hdr.index("Grid Size"), hdr.index("Block Size")
    out = []
    for r in rows[1:]:
        if r[mname] == "gpu__time_duration.sum":
            out.append((r[k], r[grid], r[blk], float(r[v]) / 1e3))
    tot = sum(x[3] for x in out) or 1.0
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); {len(out)} launches")
    print(f"# {'idx':>3} {'us':>10} {'share':>6}  grid        block      kernel")
    for i, (name, g, b, us) in enumerate(out):
        print(f"  {i:>3} {us:>10.1f} {100 * us / tot:>5.1f}%  {g:<11} {b:<10} {name}")
    agg = OrderedDict()
    for name, g, b, us in out:
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += us
    print("# per kernel: launches, total us, share")
    for name, (c, us) in agg.items():
        print(f"  {c:>4} {us:>10.1f} {100 * us / tot:>5.1f}%  {name}")


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def full(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full --clock-control none report: {path}")
    for row in rows[2:]:
        print(f"## {row[hdr.index('Kernel Name')]}")
        for m, label in WANT:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {label:<22} {row[i]:>16} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
