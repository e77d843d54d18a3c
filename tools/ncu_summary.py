"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per kernel (template-resolved) launches, mean / total time and share."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[i], rows[i + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi = hdr.index("Grid Size")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in data:
        out.append((re.sub(r"\(sr::\w+\)|\(.*", "", r[ki]).strip(),
                    float(r[vi].replace(",", "")) * scale[r[ui]], r[gi]))
    return out


def main(path, top=20):
    seq = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, set()])
    for name, us, g in seq:
        a = agg[name]
        a[0] += 1
        a[1] += us
        a[2].add(g)
    tot = sum(x[1] for x in seq)
    print(f"{'total us':>10} {'n':>5} {'us/launch':>10} {'share':>6}  kernel [grids]")
    for name, (n, t, grids) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:10.1f} {n:5d} {t / n:10.2f} {100 * t / tot:5.1f}%  {name} {sorted(grids)[:3]}")
    print(f"total {tot:.1f} us over {len(seq)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
