#!/usr/bin/env python
"""Markdown table: explicit im2col+GEMM vs implicit, per layer (time from the
CUDA-graph run of tools/overhead.py, DRAM bytes from its ncu --once pass).

  python tools/overhead_summary.py gpurun_out/overhead_cfg4.json gpurun_out/overhead_ncu_cfg4_n16.csv [more.json ...]

The ncu launch list of `overhead.py --once` is, per layer, the implicit
segment ([pad] conv) followed by the explicit one (im2col [pad] gemm-conv);
each segment ends at a conv kernel, which is how it is split here (torch
kernels that create the operands are skipped).
"""

import csv
import json
import sys


def ncu_segments(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, im, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    by, order = {}, []
    for r in rows[1:]:
        key = (r[iid], r[ik])
        if key not in by:
            by[key] = {}
            order.append(key)
        by[key][r[im]] = float(r[iv].replace(",", ""))
    segs, cur = [], []
    for key in order:
        if "imconv::" not in key[1]:      # torch kernels creating the next layer's operands
            continue
        cur.append(by[key])
        if "imconv::conv_" in key[1]:  # any conv kernel (generic / row-band / halo) ends a segment
            segs.append(cur)
            cur = []
    tot = lambda seg, m: sum(k.get(m, 0.0) for k in seg)
    out = []
    for i in range(0, len(segs) - 1, 2):
        imp, exp = segs[i], segs[i + 1]
        out.append({
            "impl_us": tot(imp, "gpu__time_duration.sum") / 1e3,
            "expl_us": tot(exp, "gpu__time_duration.sum") / 1e3,
            "impl_dram_MB": (tot(imp, "dram__bytes_read.sum") + tot(imp, "dram__bytes_write.sum")) / 1e6,
            "expl_dram_MB": (tot(exp, "dram__bytes_read.sum") + tot(exp, "dram__bytes_write.sum")) / 1e6,
            "expl_launches": len(exp),
        })
    return out


def main():
    jsons = [a for a in sys.argv[1:] if a.endswith(".json")]
    csvs = [a for a in sys.argv[1:] if a.endswith(".csv")]
    for jp in jsons:
        d = json.load(open(jp))
        rows = d["layers"]
        print(f"\n### {d['config']} (batch {d['n']} per layer, unique layers, CUDA-graph timing)\n")
        print("| layer | implicit (ms) | explicit (ms) | explicit / implicit | lowered / ifmap bytes | "
              "algorithmic MB implicit | algorithmic MB explicit | max rel diff |")
        print("|---|---|---|---|---|---|---|---|")
        for r in rows:
            print(f"| {r['layer']} | {r['implicit_ms']:.4f} | {r['explicit_ms']:.4f} | {r['slowdown']:.2f} | "
                  f"{r['lowered_over_ifmap']:.2f} | {r['alg_bytes_implicit_MB']:.1f} | "
                  f"{r['alg_bytes_explicit_MB']:.1f} | {r['max_rel_diff']:.4f} |")
        ti = sum(r["implicit_ms"] for r in rows)
        te = sum(r["explicit_ms"] for r in rows)
        ai = sum(r["alg_bytes_implicit_MB"] for r in rows)
        ae = sum(r["alg_bytes_explicit_MB"] for r in rows)
        print(f"| **total** | **{ti:.4f}** | **{te:.4f}** | **{te / ti:.2f}** | | {ai:.0f} | {ae:.0f} | |")
    for cp in csvs:
        segs = ncu_segments(cp)
        print(f"\n### ncu DRAM bytes per path (`{cp.split('/')[-1]}`, cold cache, serialised)\n")
        print("| # | implicit (us) | explicit (us) | implicit DRAM (MB) | explicit DRAM (MB) | explicit / implicit bytes |")
        print("|---|---|---|---|---|---|")
        for i, s in enumerate(segs):
            print(f"| {i} | {s['impl_us']:.1f} | {s['expl_us']:.1f} | {s['impl_dram_MB']:.1f} | "
                  f"{s['expl_dram_MB']:.1f} | {s['expl_dram_MB'] / max(s['impl_dram_MB'], 1e-9):.2f} |")
        ti = sum(s["impl_dram_MB"] for s in segs)
        te = sum(s["expl_dram_MB"] for s in segs)
        print(f"| **total** | {sum(s['impl_us'] for s in segs):.1f} | {sum(s['expl_us'] for s in segs):.1f} | "
              f"**{ti:.0f}** | **{te:.0f}** | **{te / ti:.2f}** |")


if __name__ == "__main__":
    main()
