"""Instruction count per source line of one kernel in a cubin (nvdisasm -g), to find code bloat.
usage: python scripts/sass_lines.py OBJ.o KERNEL_SUBSTRING [N]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
lines = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and pat in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith(".text.")), len(lines))
cnt, cur = collections.Counter(), None
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    elif re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+\S", l):
        cnt[cur] += 1
tot = sum(cnt.values())
print("instructions", tot)
srcs = {}
for (f, ln), c in cnt.most_common(n):
    path = next((os.path.join(r, f) for r, _, fs in os.walk("paper_2003_00822_b200") if f in fs), None)
    if path and path not in srcs:
        srcs[path] = open(path).read().splitlines()
    s = srcs[path][ln - 1].strip()[:90] if path else ""
    print(f"{c:5d}  {f}:{ln}  {s}")
