#!/usr/bin/env python
"""Summarise ncu reports / launch lists into markdown for profiles/.

  python tools/ncu_summary.py full  gpurun_out/full_*.ncu-rep      > profiles/rN/ncu_full_summary.md
  python tools/ncu_summary.py launches gpurun_out/launches.csv     > profiles/rN/launches_summary.md
"""

import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes (L2->SM)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "tensor-core smem operand reads % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % peak"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(units, r))) for r in rows[2:]]


def full(reps):
    print("| kernel / layer | " + " | ".join(n for _, n in FULL_METRICS) + " |")
    print("|---|" + "---|" * len(FULL_METRICS))
    for rep in reps:
        for rec in raw(rep):
            name = rec.get("Kernel Name", ("", "?"))[1]
            short = name.split("(")[0].replace("void ", "").replace("imconv::", "")
            cells = []
            for key, _ in FULL_METRICS:
                unit, val = rec.get(key, ("", "n/a"))
                cells.append(f"{val} {unit}".strip())
            tag = rep.split("/")[-1].replace(".ncu-rep", "")
            print(f"| {tag}: `{short}` | " + " | ".join(cells) + " |")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    by = {}
    order = []
    for r in rows[1:]:
        key = (r[hdr.index("ID")], r[ik])
        if key not in by:
            by[key] = {}
            order.append(key)
        by[key][r[im]] = float(r[iv].replace(",", ""))
    tot = sum(v.get("gpu__time_duration.sum", 0) for v in by.values())
    print(f"launches: {len(order)}, total device time {tot / 1e3:.1f} us (ncu, cold cache, serialised)\n")
    print("| # | kernel | time (us) | share | DRAM read (MB) | DRAM write (MB) |")
    print("|---|---|---|---|---|---|")
    for i, key in enumerate(order):
        v = by[key]
        t = v.get("gpu__time_duration.sum", 0)
        short = key[1].split("(")[0].replace("void ", "").replace("imconv::", "")
        rd = v.get("dram__bytes_read.sum")
        wr = v.get("dram__bytes_write.sum")
        f = lambda b: "" if b is None else f"{b / 1e6:.1f}"
        print(f"| {i} | `{short}` | {t / 1e3:.1f} | {100 * t / tot:.1f}% | {f(rd)} | {f(wr)} |")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2:])
    else:
        launches(sys.argv[2])
