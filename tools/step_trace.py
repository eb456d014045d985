"""Read the per-phase globaltimer stamps the persistent decode-step kernel
writes when SW_STEP_TRACE=<file> (eager steps), and print a phase timeline:
when every CTA was released into the phase (grid barrier passed), when the
last CTA arrived, and how long the activation producer waited.

  SW_STEP_TRACE=/tmp/st.bin python tools/step_check.py --model LLAMA_1B --batch 64 --prompt 512
  python tools/step_trace.py /tmp/st.bin
"""
import struct
import sys

import numpy as np

NAMES = ["qkv", "attn", "wo", "gu", "wd"]


def load(path):
    data = open(path, "rb").read()
    off, recs = 0, []
    while off < len(data):
        n_ph, ctas, R = struct.unpack_from("iii", data, off)
        off += 12
        n = n_ph * ctas * 8
        a = np.frombuffer(data, dtype=np.uint64, count=n, offset=off).reshape(n_ph, ctas, 8).astype(np.float64)
        off += n * 8
        recs.append((R, a))
    return recs


def report(R, a, last_layers=None):
    n_ph = a.shape[0]
    t0 = a[0, :, 0][a[0, :, 0] > 0].min()
    rel = lambda v: (v - t0) / 1e3
    lines = [f"rows={R} phases={n_ph} ctas={a.shape[1]}"]
    tot = {}
    prev_end = t0
    for p in range(n_ph):
        name = "lm" if p == n_ph - 1 else f"L{p // 5}.{NAMES[p % 5]}"
        kind = "lm" if p == n_ph - 1 else NAMES[p % 5]
        st, go, end, xw = a[p, :, 0], a[p, :, 1], a[p, :, 2], a[p, :, 3]
        w0, w1, m0, m1 = a[p, :, 4], a[p, :, 5], a[p, :, 6], a[p, :, 7]
        go_v = go[go > 0]
        release = go_v.max() if len(go_v) else np.nan
        last = end.max()
        dur = (last - prev_end) / 1e3
        tot[kind] = tot.get(kind, 0.0) + dur
        xv = xw[xw > 0]
        def med(v):
            v = v[v > 0]
            return rel(np.median(v)) if len(v) else float("nan")

        lines.append(f"{name:8s} rel {rel(release):8.1f} done {rel(last):8.1f} phase {dur:6.1f} us | med: "
                     f"x-go {med(xw):8.1f} w0 {med(w0):8.1f} w1 {med(w1):8.1f} mma0 {med(m0):8.1f} mma1 {med(m1):8.1f} "
                     f"end {med(end):8.1f}")
        prev_end = last
    lines.append("per kind: " + "  ".join(f"{k} {v:.1f} us" for k, v in tot.items()))
    return "\n".join(lines)


if __name__ == "__main__":
    recs = load(sys.argv[1])
    for R, a in recs[-1:]:
        print(report(R, a))
