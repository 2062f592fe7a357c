"""Instruction counts of the HMMA loops of the attention kernels (nvdisasm -g output of
decode_two.o): a quick guard against register-allocation drift in the gather/dequant loop.

    python tools/mma_loops.py [paper_2603_14224_b200/_build/decode_two.o]
"""
import os
import re
import subprocess
import sys
import tempfile

obj = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "paper_2603_14224_b200", "_build", "decode_two.o")
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cubin = next(os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin"))
    L = subprocess.run(["nvdisasm", "-g", cubin], check=True, capture_output=True, text=True).stdout.splitlines()
for i0, line in enumerate(L):
    if not (line.startswith(".text.") and "decode_attend_kernel" in line):
        continue
    e = next((i for i in range(i0 + 1, len(L)) if L[i].startswith(".text.")), len(L))
    seg = L[i0:e]
    labels = {m.group(1): i for i, s in enumerate(seg) if (m := re.match(r"(\.L_x_\d+):", s))}
    loops = []
    for i, s in enumerate(seg):
        m = re.search(r"BRA `\((\.L_x_\d+)\)", s)
        if m and m.group(1) in labels and labels[m.group(1)] < i:
            body = seg[labels[m.group(1)]:i + 1]
            n = sum(1 for b in body if re.match(r"\s+/\*[0-9a-f]{4,6}\*/", b))
            if any("HMMA" in b for b in body):
                loops.append(n)
    print(re.search(r"decode_attend_kernel\w*", line).group(0), loops)
