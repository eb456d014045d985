"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        out.append((r[ki], v))
    return out


def summary(path, top=16):
    launches = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in launches:
        key = name.split("(")[0][:80]
        agg[key][0] += 1
        agg[key][1] += us
    total = sum(v for _, v in launches)
    lines = [f"{path}: {len(launches)} launches, {total:.1f} us total (serialised, cold cache)"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{v:10.1f} us {100 * v / total:5.1f}% {n:5d}x {v / n:9.2f} us  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
