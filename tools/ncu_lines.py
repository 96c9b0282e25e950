"""Aggregate ncu warp-stall samples of a kernel by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL [top]

Maps SASS offsets to source lines with `nvdisasm -g` on the library's cubin
(needs -lineinfo) and sums the "Warp Stall Sampling (All Samples)" column of
`ncu --page source --print-source sass`.
"""

from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_map(lib: str, kernel: str) -> dict:
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub[0])], capture_output=True, text=True).stdout
    m, cur, inside = {}, None, False
    for ln in out.splitlines():
        if ln.startswith(".text."):
            name = ln.strip()[6:-1]
            inside = name == kernel or (kernel in name and not name.startswith("$"))
            continue
        if not inside:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = f"{os.path.basename(g.group(1))}:{g.group(2)}"
            continue
        g = re.match(r"\s+/\*([0-9a-f]+)\*/", ln)
        if g and cur:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    rep, lib, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kernel], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    excl = os.environ.get("EXCLUDE", "stall_barrier").split(",")
    recs = []
    for r in rows[hi + 1:]:
        if len(r) <= iss or not r[ia].startswith("0x"):
            continue
        per = {hdr[i]: int(r[i] or 0) for i in reasons}
        tot = int(r[iss] or 0) - sum(per[e] for e in excl if e in per)
        recs.append((int(r[ia], 16), tot, per))
    base = min(a for a, _, _ in recs)
    lm = line_map(lib, kernel)
    agg = collections.Counter()
    why = collections.defaultdict(collections.Counter)
    for a, s, per in recs:
        k = lm.get(a - base, "?")
        agg[k] += s
        for rn, v in per.items():
            if rn not in excl:
                why[k][rn] += v
    tot = sum(agg.values())
    src = {}
    for k, s in agg.most_common(top):
        f, _, n = k.partition(":")
        if f not in src:
            path = os.path.join(os.path.dirname(os.path.abspath(lib)), "csrc", f)
            src[f] = open(path).read().splitlines() if os.path.exists(path) else []
        line = src[f][int(n) - 1].strip() if n.isdigit() and int(n) <= len(src[f]) else ""
        top2 = ",".join(f"{n[6:]}:{v * 100 // max(s, 1)}" for n, v in why[k].most_common(2))
        print(f"{s:8d} {100 * s / tot:5.1f}%  {k:22s} {top2:28s} {line[:70]}")


if __name__ == "__main__":
    main()
