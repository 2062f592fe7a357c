"""Per-source-line dynamic instruction counts and stall samples of one kernel: joins an ncu
source page (--page source --csv --print-source sass) with nvdisasm -g line info by
instruction order.

    python tools/sass_line_profile.py ncu_source.csv nvdisasm_g.sass <mangled kernel> [N]
"""
import collections
import csv
import re
import sys

src, dis, name = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(src)))
hdr = rows[1]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
L = open(dis).read().splitlines()
s = next(i for i, l in enumerate(L) if l.startswith(".text." + name))
e = next((i for i in range(s + 1, len(L)) if L[i].startswith(".text.")), len(L))
lines, cur = [], None
for l in L[s:e]:
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+\S", l):
        lines.append(cur)
assert len(lines) >= len(data), (len(lines), len(data))
cnt, smp, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for ln, r in zip(lines, data):
    n = int(r[ie] or 0)
    cnt[ln] += n
    smp[ln] += int(r[ss] or 0)
    ops[ln][r[1].split()[0].lstrip("@!P0123456789U ").split(".")[0] if r[1].split() else "?"] += n
T, S = sum(cnt.values()), sum(smp.values())
print(f"warp instructions {T}, stall samples {S}")
for ln, n in cnt.most_common(top):
    print(f"{ln:18s} {n / T:6.1%} inst  {smp[ln] / S:6.1%} samples  {ops[ln].most_common(4)}")
