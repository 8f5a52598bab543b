"""Annotated hot SASS of one device function: address, executions, stall samples, source line, instruction.

usage: python tools/hot_sass.py DISASM_G.txt NCU_SASS.csv FUNC_SUBSTR MIN_EXEC
"""
import csv
import re
import sys

dis, sass, want, mn = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text._ZN6slosim10sim_kernel")][0]
fn, cur, amap = "sim_kernel", None, {}
for l in lines[start:]:
    if l.startswith("//---------------------") and amap:
        break
    m = re.search(r"\.type\s+\$\S*?\$(\S+),@function", l)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
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
cols = [c for c in ("stall_wait", "stall_long_sb", "stall_short_sb", "stall_no_inst", "stall_branch_resolving") if c in hdr]
base = int(rows[0][0], 16)
for r in rows:
    a = int(r[0], 16) - base
    e = int(r[ie] or 0)
    f, ln = amap.get(a, ("?", "?"))
    if want in f and e >= mn:
        st = " ".join(f"{c[6:]}={r[hdr.index(c)]}" for c in cols if r[hdr.index(c)] not in ("0", ""))
        print(f"{a:6x} {e / 1e6:7.2f}M {int(r[isamp] or 0):6d} {str(ln):18s} {r[1].strip()[:64]:64s} {st}")
