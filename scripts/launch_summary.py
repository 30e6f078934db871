"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/launch_summary.py launches.csv [title] > summary.md
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    acc = OrderedDict()
    for r in rows[1:]:
        name = r[kn].replace("(int)", "").split("(")[0].replace("void ", "")
        ms = float(r[mv].replace(",", "")) * scale.get(r[mu], 1e-6)
        n, t = acc.get(name, (0, 0.0))
        acc[name] = (n + 1, t + ms)
    total = sum(t for _, t in acc.values())
    print(f"# ncu launch list {title} (pass kernels; serialised, cold-cache)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for name, (n, t) in acc.items():
        print(f"| {name} | {n} | {t:.2f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    main()
