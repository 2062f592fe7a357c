"""Per-CUDA-line stall samples and executed instructions from
`ncu --page source --csv --print-source cuda,sass`."""
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
        n = float(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    out.append((s, n, fname, r[0], r[1]))
tot = sum(x[0] for x in out)
ntot = sum(x[1] for x in out)
print(f"total samples {tot:.0f}, warp-instructions {ntot:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
for s, ni, f, ln, src in sorted(out, key=lambda x: -x[key])[:n]:
    print(f"{100*s/tot:5.1f}% {100*ni/ntot:5.1f}%i {f}:{ln:5s} {src.strip()[:95]}")
