"""Per-source-line samples / executed instructions / stall columns from
`ncu --page source --csv --print-source cuda,sass` (CUDA-level rows only).

    python tools/ncu_src.py report_src.csv [N] [inst|samples] [--ranges]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "samples"
rows = csv.reader(open(path))
fname, hdr = "", None
recs = []
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
        ni = float(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError, KeyError):
        continue
    stalls = {h: float(r[i] or 0) for h, i in hdr.items() if h.startswith("stall_") and "Not Issued" not in h
              and r[i] not in ("", "-")}
    recs.append((fname, int(r[0]), r[1], s, ni, stalls))
ts = sum(x[3] for x in recs)
ti = sum(x[4] for x in recs)
print(f"total samples {ts:.0f}, warp-instructions {ti:.0f}")
k = 4 if key == "inst" else 3
for f, ln, src, s, ni, st in sorted(recs, key=lambda x: -x[k])[:n]:
    top = sorted(st.items(), key=lambda x: -x[1])[:2]
    tops = " ".join(f"{a[6:]}={b:.0f}" for a, b in top)
    print(f"{100*s/ts:5.1f}% {100*ni/ti:5.1f}%i {f}:{ln:<5d} {src.strip()[:70]:70s} {tops}")

if "--ranges" in sys.argv:
    # decode_common.cuh regions (edit when the file moves)
    regions = [("table build", "decode_common.cuh", 14, 70), ("score_batch", "decode_common.cuh", 71, 200),
               ("attention", "decode_common.cuh", 240, 570), ("geom/sample load", "decode_common.cuh", 571, 634),
               ("B1 sample/tau", "decode_common.cuh", 635, 771), ("B2 loop+append", "decode_common.cuh", 772, 841),
               ("exact fallback", "decode_common.cuh", 842, 876), ("select/emit", "decode_common.cuh", 877, 1100)]
    agg = defaultdict(lambda: [0.0, 0.0])
    for f, ln, src, s, ni, st in recs:
        name = f
        for rn, rf, a, b in regions:
            if f == rf and a <= ln <= b:
                name = rn
        agg[name][0] += s
        agg[name][1] += ni
    for name, (s, ni) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {name:24s} samples {100*s/ts:5.1f}%  inst {100*ni/ti:5.1f}%")
