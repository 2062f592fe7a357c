"""Static SASS instruction count per source line of one kernel (nvdisasm --print-line-info
output), to spot rematerialised or duplicated code in hot loops.

    nvcc ... -lineinfo -cubin -o k.cubin file.cu && nvdisasm --print-line-info k.cubin > k.sass
    python tools/sass_lines.py k.sass decode_select_kernel decode_common.cuh 780-835 85-100
"""
import collections
import re
import sys

path, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = [tuple(int(v) for v in r.split("-")) for r in sys.argv[4:]]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//-----") and ".text" in lines[i]),
           len(lines))
cur, cnt = None, collections.Counter()
for l in lines[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,6}\*/", l):
        cnt[cur] += 1
print(f"{kern}: {sum(cnt.values())} instructions")
src = None
for (f, ln), c in sorted(cnt.items(), key=lambda x: (x[0][0] or "", x[0][1])):
    if f == fname and any(a <= ln <= b for a, b in ranges):
        if src is None:
            src = open("paper_2603_14224_b200/csrc/" + fname).read().splitlines()
        print(f"{ln:5d} {c:5d}  {src[ln - 1].strip()[:90]}")
