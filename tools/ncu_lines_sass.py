"""Per-source-line totals of an ncu SASS source page (instructions, thread instructions, stall samples).

usage: python tools/ncu_lines_sass.py DISASM_G.txt NCU_SASS.csv KERNEL_SUBSTR [top]
(DISASM_G: nvdisasm -c -g of the profiled cubin; NCU_SASS: ncu -i REP --page source --csv --print-source sass)
"""
import csv
import re
import sys
from collections import defaultdict

dis, sass, want = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and want in l][0]
cur, amap = None, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        if amap:
            break
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass)))
hdr = rows[1]
ie, ti, ns = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0, 0])
base = None
for r in rows[2:]:
    if not r or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    ln = amap.get(a - base, "?")
    agg[ln][0] += int(r[ie] or 0)
    agg[ln][1] += int(r[ti] or 0)
    agg[ln][2] += int(r[ns] or 0)
tot = [sum(v[k] for v in agg.values()) for k in range(3)]
print(f"total inst {tot[0]:.3e} thread-inst {tot[1]:.3e} (lanes/inst {tot[1] / max(tot[0], 1):.2f}) samples {tot[2]}")
src = {}
for ln, (i, t, s) in sorted(agg.items(), key=lambda x: -x[1][2])[:top]:
    f, n = (ln.split(":") + ["0"])[:2]
    try:
        if f not in src:
            import os
            p = next(p for p in [f"paper_2605_02329_b200/csrc/{f}", f"include/{f}"] if os.path.exists(p))
            src[f] = open(p).read().split("\n")
        text = src[f][int(n) - 1].strip()[:80]
    except Exception:
        text = ""
    print(f"{100 * s / tot[2]:5.1f}% smp {100 * i / tot[0]:5.1f}% inst  lanes {t / max(i, 1):5.1f}  {ln:18s} {text}")
