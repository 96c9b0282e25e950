"""Local-memory (spill) instructions of a kernel by CUDA source line.

    python tools/spill_lines.py [LIB.so] [KERNEL]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2508_06041_b200/libdpq_b200.so"
kernel = sys.argv[2] if len(sys.argv) > 2 else "engine_kernel"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
inside, cur, res = False, None, collections.Counter()
for ln in out.splitlines():
    if ln.startswith(".text."):
        inside = ln.strip()[6:-1] == kernel
        continue
    if not inside:
        continue
    g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if g:
        cur = f"{os.path.basename(g.group(1))}:{g.group(2)}"
        continue
    m = re.search(r"\b(LDL|STL)(\.\w+)*\b", ln)
    if m:
        res[(cur, m.group(1))] += 1
srcs = {}
for (c, op), n in sorted(res.items(), key=lambda x: (x[0][0] or "", x[0][1])):
    f, l = c.split(":")
    path = os.path.join(os.path.dirname(lib), "csrc", f)
    if path not in srcs:
        srcs[path] = open(path).read().splitlines() if os.path.exists(path) else []
    txt = srcs[path][int(l) - 1].strip()[:90] if srcs[path] else ""
    print(f"{op} {n:3d} {c:28s} {txt}")
