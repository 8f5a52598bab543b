"""Executed instructions / stall samples per device function (inlined code attributed to its source function).

usage: python tools/func_exec.py DISASM_G.txt NCU_SASS.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict

dis, sass = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text._ZN6slosim10sim_kernel")][0]
cur, amap = None, {}
for l in lines[start:]:
    if l.startswith("//---------------------") and amap:
        break
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s", l)
    if m:
        amap[int(m.group(1), 16)] = cur
defs = {}
for f in ("engine.cuh", "lut.cuh", "numerics.cuh"):
    d = []
    for i, l in enumerate(open(f"paper_2605_02329_b200/csrc/{f}").read().split("\n"), 1):
        m = re.match(r"^(?:template\s*<.*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\s*\(", l)
        if m and not l.rstrip().endswith(";"):
            d.append((i, m.group(1)))
    defs[f] = d
hdr, rows = None, []
for r in csv.reader(open(sass)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if r and r[0].startswith("0x"):
        rows.append(r)
ie, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[0][0], 16)
agg = defaultdict(lambda: [0, 0])
for r in rows:
    loc = amap.get(int(r[0], 16) - base)
    name = "?"
    if loc:
        name = loc[0]
        for i, n in defs.get(loc[0], []):
            if i <= loc[1]:
                name = n
    agg[name][0] += int(r[ie] or 0)
    agg[name][1] += int(r[isamp] or 0)
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, (e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * e / te:5.1f}% exec {100 * s / ts:5.1f}% samples  {k}")
