"""Innermost SASS loops of a kernel with their instruction mix (nvdisasm --print-line-info
output).  Used to find per-batch overhead in the selection kernel's scoring loop.

    python tools/sass_loops.py k.sass decode_select_kernel [min_FADD2]
"""
import collections
import re
import sys

path, kern = sys.argv[1], sys.argv[2]
minf = int(sys.argv[3]) if len(sys.argv) > 3 else 50
L = open(path).read().splitlines()
s = next(i for i, l in enumerate(L) if l.startswith(".text.") and kern in l)
e = next((i for i in range(s + 1, len(L)) if L[i].startswith(".text.")), len(L))
seg = L[s:e]
labels = {}
for i, l in enumerate(seg):
    m = re.match(r"(\.L_x_\d+):", l)
    if m:
        labels[m.group(1)] = i
loops = []
for i, l in enumerate(seg):
    m = re.search(r"BRA `\((\.L_x_\d+)\)", l)
    if m and m.group(1) in labels and labels[m.group(1)] < i:
        body = seg[labels[m.group(1)]:i + 1]
        ops = collections.Counter()
        for b in body:
            mm = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", b)
            if mm:
                ops[mm.group(3) + ("" if mm.group(3) != "IMAD" else (mm.group(4) or ""))] += 1
        if ops["FADD2"] >= minf:
            loops.append((sum(ops.values()), m.group(1), ops))
for n, lab, ops in sorted(loops)[:3]:
    print(lab, n, ops.most_common(30))
