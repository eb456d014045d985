"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optionally with
dram__bytes_read.sum / dram__bytes_write.sum): per kernel, total and per-launch
time, share of the list, and DRAM bytes / achieved GB/s when captured."""
import collections
import csv
import sys

UNIT_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
UNIT_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    """[(kernel name, us, dram bytes or None)] in launch order."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(r[ii], {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            d["us"] = v * UNIT_US.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            d["bytes"] = d.get("bytes", 0.0) + v * UNIT_B.get(r[ui], 1.0)
    return [(d["name"], d["us"], d.get("bytes")) for d in per.values() if "us" in d]


def summary(path, top=16):
    launches = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for name, us, b in launches:
        key = name.split("(")[0].replace("(anonymous namespace)::", "")[:80]
        a = agg[key]
        a[0] += 1
        a[1] += us
        a[2] += b or 0.0
    total = sum(v for _, v, _ in launches)
    lines = [f"{path}: {len(launches)} launches, {total:.1f} us total (serialised, cold cache)"]
    for k, (n, v, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        extra = f"  {b / n / 1e6:9.1f} MB/launch {b / v / 1e3:8.1f} GB/s DRAM" if b else ""
        lines.append(f"{v:10.1f} us {100 * v / total:5.1f}% {n:5d}x {v / n:9.2f} us{extra}  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
