"""Registers / spills per kernel from build.log (nvcc -Xptxas -v): python tools/ptxas_summary.py [regex]"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
log = open("paper_2509_19777_b200/build.log").read().splitlines()
name = None
for i, l in enumerate(log):
    m = re.search(r"Compiling entry function '(\w+)'", l)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        spill = regs = ""
        for l2 in log[i + 1:i + 4]:
            if "spill" in l2:
                spill = re.sub(r".*?(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads.*",
                               r"stack \1 st \2 ld \3", l2)
            if "registers" in l2:
                regs = re.sub(r".*Used (\d+) registers.*", r"\1 regs", l2)
        if pat.search(name):
            print(f"{regs:9s} {spill:24s} {name[:150]}")
