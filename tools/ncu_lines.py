"""Per-CUDA-line stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out = []
fname = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r or r[0] in ("", "Function Name"):
        continue
    try:
        s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    out.append((s, fname, r[0], r[1]))
tot = sum(x[0] for x in out)
print("total", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, f, ln, src in sorted(out, key=lambda x: -x[0])[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src.strip()[:100]}")
