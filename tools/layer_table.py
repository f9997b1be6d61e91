#!/usr/bin/env python
"""Per-layer table from an ncu launch list of one bench step (53 launches, in
resnet50_layers order): device time, DRAM bytes, roofline fraction.

  python tools/layer_table.py gpurun_out/launches.csv [--group] [--n 32]

--n: the per-GPU batch the launch list was taken at (an emulated shard), default 256.
"""
import csv
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

from paper_2110_03901_b200.lowering import touched_pixels  # noqa: E402
from paper_2110_03901_b200.workloads import resnet50_layers  # noqa: E402

PEAK_TF, HBM = 1412.1, 6550.4  # MEASURED_PEAKS.json (bf16 sustained, copy GB/s)


def main(path, group, n=256):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iid, im, iv = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    order = []
    for r in rows[1:]:
        if r[iid] not in per:
            per[r[iid]] = {}
            order.append(r[iid])
        per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
    layers = resnet50_layers(n)
    assert len(order) == len(layers), (len(order), len(layers))
    agg = {}
    tot_t = tot_roof = tot_traffic = tot_alg = 0.0
    print("| layer | us | TFLOP/s | alg MB | DRAM MB | roofline frac |")
    print("|---|---|---|---|---|---|")
    for lid, layer in zip(order, layers):
        sp = layer.spec
        m = per[lid]
        t = m["gpu__time_duration.sum"] / 1e3
        alg = sp.n * touched_pixels(sp) * sp.c_i * 2 + sp.h_f * sp.w_f * sp.c_i * sp.c_o * 2 + sp.gemm_m * sp.c_o * 2
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        roof = max(sp.flops / (PEAK_TF * 1e12), alg / (HBM * 1e9)) * 1e6
        tot_t += t
        tot_roof += roof
        tot_traffic += dram
        tot_alg += alg
        key = (layer.name[:2], layer.name.split("_")[-1])
        a = agg.setdefault(key, [0, 0, 0, 0])
        a[0] += t
        a[1] += roof
        a[2] += 1
        a[3] += sp.flops
        if not group:
            print(f"| {layer.name} | {t:.1f} | {sp.flops / t / 1e6:.0f} | {alg / 1e6:.1f} | {dram / 1e6:.1f} | "
                  f"{roof / t:.2f} |")
    if group:
        for k, (t, roof, c, f) in sorted(agg.items(), key=lambda x: -(x[1][0] - x[1][1])):
            print(f"| {k[0]} {k[1]} (x{c}) | {t:.1f} | {f / t / 1e6:.0f} | | | {roof / t:.2f} |")
    flops = sum(l.spec.flops for l in layers)
    print(f"\ntotal {tot_t:.1f} us ({flops / tot_t / 1e6:.0f} TFLOP/s), roofline {tot_roof:.1f} us "
          f"(frac {tot_roof / tot_t:.2f}); DRAM traffic {tot_traffic / 1e9:.2f} GB vs algorithmic "
          f"{tot_alg / 1e9:.2f} GB ({tot_traffic / tot_alg:.2f}x)")


if __name__ == "__main__":
    argv = sys.argv[1:]
    n = int(argv[argv.index("--n") + 1]) if "--n" in argv else 256
    main(argv[0], "--group" in argv, n)
