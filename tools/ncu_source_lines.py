"""Per-CUDA-source-line hot spots of an ncu --set full --import-source report
(compiled with -lineinfo): warp-stall samples, instructions executed and the
dominant stall reasons per line.
usage: python tools/ncu_source_lines.py <report.ncu-rep> [top=25]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name") and len(r) == len(hdr):
        lines.append((fname, r))
if not hdr:
    sys.exit("no source page")
ix = {k: i for i, k in enumerate(hdr)}
stalls = [k for k in hdr if k.startswith("stall_")]
tot_s = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for _, r in lines)
tot_i = sum(float(r[ix["Instructions Executed"]] or 0) for _, r in lines)
lines.sort(key=lambda fr: -float(fr[1][ix["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
print(f"{'file:line':22s} {'samp%':>6s} {'inst%':>6s}  top stalls | source")
for f, r in lines[:top]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ins = float(r[ix["Instructions Executed"]] or 0)
    st = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    sts = " ".join(f"{n}:{100 * v / max(s, 1):.0f}" for v, n in st if v > 0)
    print(f"{f + ':' + r[0]:22s} {100 * s / tot_s:6.1f} {100 * ins / tot_i:6.1f}  {sts:34s} | {r[1].strip()[:70]}")
