"""Development aid: count STL/LDL (stack traffic) per source line of one kernel in an object file.
    python scripts/spills.py <file.o> <kernel-name-substring>"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
               capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True,
                      text=True).stdout
cur_fn, cur_line, cnt = None, None, collections.Counter()
for l in sass.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur_fn = m.group(1)
    m = re.search(r'File "(?:.*/)?([^/"]+)", line (\d+)', l)
    if l.strip().startswith("//##") and m:
        cur_line = f"{m.group(1)}:{m.group(2)}"
    if cur_fn and pat in cur_fn and re.search(r"\b(STL|LDL)", l):
        cnt[(cur_line, "STL" if "STL" in l else "LDL")] += 1
for (line, op), n in sorted(cnt.items(), key=lambda x: str(x[0])):
    print(f"{line}: {op} x{n}")
print("total", sum(cnt.values()))
