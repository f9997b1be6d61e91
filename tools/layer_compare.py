#!/usr/bin/env python
"""Compare two bench.py --layers-json files grouped by layer type.

  python tools/layer_compare.py old.json new.json
"""
import collections
import json
import sys


def grouped(path):
    d = json.load(open(path))
    g = collections.OrderedDict()
    for l in d["layers"]:
        name = l["layer"]
        key = name[:2] + " " + name.split("_", 1)[1] if "_" in name else name
        e = g.setdefault(key, [0.0, 0.0, 0])
        e[0] += l["ms"]
        e[1] += l["ms"] * l["roofline_frac"]
        e[2] += 1
    return d, g


def main():
    da, ga = grouped(sys.argv[1])
    db, gb = grouped(sys.argv[2])
    print(f"| group | n | old (us) | new (us) | roofline (us) | frac |")
    print("|---|---|---|---|---|---|")
    for k, (ms, roof, n) in sorted(gb.items(), key=lambda kv: -(kv[1][0] - kv[1][1])):
        print(f"| {k} | {n} | {ga.get(k, [0])[0] * 1e3:.1f} | {ms * 1e3:.1f} | {roof * 1e3:.1f} | {roof / ms:.2f} |")
    print(f"\nstep kernel time: old {da['kernel_ms']:.4f} ms, new {db['kernel_ms']:.4f} ms; "
          f"roofline {db['roofline_ms']:.4f} ms (frac {db['roofline_ms'] / db['kernel_ms']:.3f})")


if __name__ == "__main__":
    main()
