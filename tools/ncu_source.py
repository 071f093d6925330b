"""Top CUDA source lines by warp-stall samples from an ncu report (-lineinfo build).

    python tools/ncu_source.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
data, fname, hdr = [], "?", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or len(r) != len(hdr):
        continue
    try:
        w = float(r[4] or 0)
        nw = float(r[5] or 0)
    except ValueError:
        continue
    data.append((w, nw, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot:.0f}")
for w, nw, loc, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * w / tot:5.1f}% (not-issued {100 * nw / tot:5.1f}%)  {loc:>22}  {src}")
