"""Per-kernel SASS opcode summary of the shipped library (cuobjdump -sass):
the instructions that prove the Blackwell paths (UTCHMMA/UTCQMMA = tcgen05.mma,
UTMALDG = TMA tensor load, LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit),
plus the warp-level MMA (HMMA) and global-load mix.

  python tools/sass_summary.py paper_2505_03763_b200/libsplitwise.so > profiles/r02/sass_summary.txt
"""
import collections
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTCHMMA.2CTA", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "UTCBAR", "HMMA", "LDSM",
        "MUFU.EX2", "LDG.E.128", "LDG.E.ENL2.256", "STG.E.128", "SYNCS", "ELECT"]


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            kernels[cur]["_total"] += 1
            if op.startswith("UTCHMMA.2CTA"):
                kernels[cur]["UTCHMMA.2CTA"] += 1
                continue
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    kernels[cur][k] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
    print(f"# SASS opcode counts per kernel of {path} (cuobjdump -sass; static instruction counts)")
    for (name, c), dn in zip(kernels.items(), demangled):
        short = re.sub(r"\(.*", "", dn.replace("(anonymous namespace)::", ""))[:110]
        ops = ", ".join(f"{k} {c[k]}" for k in KEYS if c[k])
        print(f"{c['_total']:6d} instr  {short}\n         {ops or '-'}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2505_03763_b200/libsplitwise.so")
