"""Per-shape mean GPU time from an ncu launch list of tools/gemm_sweep.py."""
import collections
import csv
import sys

NAMES = ["1b.qkv", "1b.wo", "1b.gu", "1b.wd", "1b.lm", "8b.qkv", "8b.wo", "8b.gu", "8b.wd"]
BYTES = {"1b.qkv": 3072 * 2048 * 2, "1b.wo": 2048 * 2048 * 2, "1b.gu": 16384 * 2048 * 2, "1b.wd": 2048 * 8192 * 2,
         "1b.lm": 128256 * 2048 * 2, "8b.qkv": 6144 * 4096 * 2, "8b.wo": 4096 * 4096 * 2, "8b.gu": 28672 * 4096 * 2,
         "8b.wd": 4096 * 14336 * 2}
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    by = collections.OrderedDict()
    for r in rows[1:]:
        if "gemm_tc" in r[ki] and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
            by[r[ii]] = v
    t = list(by.values())
    out = []
    for si, n in enumerate(NAMES):
        seg = t[si * 38:(si + 1) * 38][8:]
        us = sum(seg) / len(seg)
        out.append(f"{n}:{us:.1f}us/{BYTES[n] / us / 1e3:.0f}GB/s")
    print(f, " ".join(out))
