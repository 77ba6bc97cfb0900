"""Per-kernel SASS opcode summary of the built library (no GPU needed):
TMA bulk copies (UBLKCP), bulk L2 prefetches (UBLKPF), FP64 tensor-core MMA
(DMMA), FP64 FMA (DFMA), mbarrier ops (SYNCS*), shared / global loads.

usage: python tools/sass_summary.py [out.txt]   (reads paper_2509_19777_b200/build/*.o)
"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UBLKCP", "UBLKPF", "DMMA", "DFMA", "SYNCS", "LDS", "LDG", "STG", "SHFL", "BAR"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.split("\n")


def main():
    rows = []
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2509_19777_b200", "build", "*.cu.o"))):
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        cur, counts = None, {}
        for line in sass.split("\n"):
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                cur = m.group(1)
                counts[cur] = collections.Counter()
                continue
            if cur is None:
                continue
            m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                op = m.group(1)
                for k in OPS:
                    if op.startswith(k):
                        counts[cur][k] += 1
        names = list(counts)
        for n, d in zip(names, demangle(names)):
            c = counts[n]
            if any(c[k] for k in ("UBLKCP", "UBLKPF", "DMMA")) or "k_sn_solve" in d or "k_ebe" in d:
                rows.append((os.path.basename(obj), d.split("(")[0].replace("hplmm::", ""), c))
    lines = ["# SASS opcode counts per kernel (cuobjdump -sass of the sm_100a objects; static "
             "instruction counts, not executions)",
             "object".ljust(18) + "kernel".ljust(48) + "".join(k.rjust(8) for k in OPS)]
    for obj, name, c in rows:
        lines.append(obj.ljust(18) + name[:47].ljust(48) + "".join(str(c[k]).rjust(8) for k in OPS))
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
