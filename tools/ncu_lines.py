"""Aggregate an ncu source-page export (cuda,sass) per CUDA source line and per function.

usage: python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
cur = None
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] == "File Path":
        cur = rec[1]
        continue
    if rec[0].isdigit():
        try:
            samples = int(rec[4]); inst = int(rec[7])
        except ValueError:
            continue
        rows.append((cur, int(rec[0]), rec[1].strip(), samples, inst))
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print(f"total samples {tot_s}  total warp-inst {tot_i:.3e}")
# function map: nearest preceding definition line in each file
funcs = {}
for f in {r[0] for r in rows}:
    try:
        src = open(f).read().splitlines()
    except OSError:
        continue
    defs = []
    for i, line in enumerate(src, 1):
        m = re.match(r"^(?:template\s*<.*>\s*)?(?:static\s+)?(?:__device__|__global__|__host__).*?(\w+)\s*\(", line)
        if m and not line.rstrip().endswith(";"):
            defs.append((i, m.group(1)))
        m2 = re.match(r"^\s{0,4}(?:__device__\s+)?(?:__forceinline__\s+|__noinline__\s+)?[\w:<>]+\s+(\w+)\s*\(.*\)\s*(const\s*)?\{?\s*$", line)
        if m2 and line.startswith("  ") and "Sim" in f and False:
            defs.append((i, m2.group(1)))
    funcs[f] = defs
agg = {}
for f, ln, s, smp, ins in rows:
    name = "?"
    for i, n in funcs.get(f, []):
        if i <= ln:
            name = n
    k = (f.split("/")[-1], name)
    a = agg.setdefault(k, [0, 0])
    a[0] += smp; a[1] += ins
print("\n== per function (by enclosing top-level definition) ==")
for k, (smp, ins) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{smp / tot_s * 100:6.2f}% samp {ins / tot_i * 100:6.2f}% inst  {k[0]}:{k[1]}")
print("\n== per line ==")
for f, ln, s, smp, ins in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{smp / tot_s * 100:6.2f}% samp {ins / tot_i * 100:6.2f}% inst  {f.split('/')[-1]}:{ln}  {s[:90]}")
