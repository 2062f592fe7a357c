"""Per-kernel SASS opcode histogram of libsikv_b200.so (cuobjdump -sass): the evidence of which
hardware paths each kernel uses (HMMA = mma.sync tensor cores, F2FP...E2M1 = e2m1 unpack,
FADD2 = packed fp32 adds, LDGSTS = cp.async, UBLKCP / UTMALDG = TMA, SYNCS = mbarriers,
REDUX / MATCH = warp reductions, DFMA = fp64).

    python tools/sass_opcodes.py [lib.so] > profiles/round2/sass_opcodes.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_14224_b200/libsikv_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern, hist = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        hist[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and kern:
        hist[kern][m.group(2)] += 1
KEY = ("HMMA", "UTCHMMA", "UTCQMMA", "F2FP", "FADD2", "FFMA2", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "LDS", "STS",
       "LDG", "STG", "PRMT", "DFMA", "MUFU", "REDUX", "MATCH", "SHFL", "BAR", "ATOMS", "ATOMG")
demangle = subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True, text=True).stdout.splitlines()
for (k, h), name in sorted(zip(hist.items(), demangle), key=lambda x: -sum(x[0][1].values())):
    fam = collections.Counter()
    for op, n in h.items():
        base = op.split(".")[0]
        fam[base] += n
        if op.startswith("F2FP") and "E2M1" in op:
            fam["F2FP.E2M1"] += n
    keyed = ", ".join(f"{x} {fam[x]}" for x in KEY + ("F2FP.E2M1",) if fam[x])
    print(f"{name[:90]}\n    {sum(h.values())} instructions; {keyed}")
