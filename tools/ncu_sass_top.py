"""Summarise an `ncu --page source --print-source sass --csv` dump: top stalled instructions
and stall totals by reason."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
tot = 0
reasons = {}
recs = []
for r in data:
    try:
        s = float(r[samp] or 0)
    except ValueError:
        continue
    tot += s
    recs.append((s, r[ix["Address"]], r[ix["Source"]], r))
    for h, i in ix.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                reasons[h] = reasons.get(h, 0) + float(r[i] or 0)
            except ValueError:
                pass
print("total samples", tot)
for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {v:10.0f} {100*v/max(tot,1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("top instructions:")
for s, a, src, r in sorted(recs, key=lambda x: -x[0])[:n]:
    top = sorted(((float(r[i] or 0), h) for h, i in ix.items() if h.startswith("stall_") and "Not Issued" not in h), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {a} {src[:60]:60s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
