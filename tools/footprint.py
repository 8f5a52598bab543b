"""Touched-code footprint per source line (i-cache study).

usage: python tools/footprint.py DISASM_G.txt NCU_SASS.csv FUNC_SUBSTR [top]
DISASM_G: nvdisasm -c -g of the cubin (line info); NCU_SASS: ncu --page source --csv --print-source sass.
Prints, for the named device function, the SASS instructions executed at least once per source line,
their executions and stall samples.
"""
import csv
import re
import sys
from collections import defaultdict

dis, sass, want = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text._ZN6slosim10sim_kernel")][0]
fn, cur = "sim_kernel", None
amap = {}
for l in lines[start:]:
    if l.startswith("//---------------------") and amap:
        break
    m = re.search(r"\.type\s+\$\S*?\$(\S+),@function", l)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s", l)
    if m:
        amap[int(m.group(1), 16)] = (fn, cur)
hdr, rows = None, []
for r in csv.reader(open(sass)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if r and r[0].startswith("0x"):
        rows.append(r)
ie, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[0][0], 16)
agg = defaultdict(lambda: [0, 0, 0])
tot_n = 0
for r in rows:
    a = int(r[0], 16) - base
    f, ln = amap.get(a, ("?", None))
    if want not in f:
        continue
    e = int(r[ie] or 0)
    if e == 0:
        continue
    tot_n += 1
    g = agg[ln]
    g[0] += 1; g[1] += e; g[2] += int(r[isamp] or 0)
print(f"{tot_n} executed instructions ({tot_n * 16 / 1024:.1f} KB) in {want}")
src = {}
for ln, (n, e, smp) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if ln is None:
        print(n, e, smp, "?")
        continue
    f, k = ln
    if f not in src:
        import os
        p = next((p for p in [f"paper_2605_02329_b200/csrc/{f}", f"include/{f}"] if os.path.exists(p)), None)
        src[f] = open(p).read().split("\n") if p else []
    text = src[f][k - 1].strip()[:90] if k - 1 < len(src[f]) else ""
    print(f"{n:4d} instr {e / 1e6:9.1f}M exec {smp:7d} samp  {f}:{k}  {text}")
