"""SASS size per source line inside one device function of the engine (code-footprint study).

usage: python tools/sass_lines.py CUBIN_DISASM_WITH_LINEINFO FUNC_SUBSTRING [top]
(make the input with: cuobjdump -xelf all lib.so; nvdisasm -c -g capi.sm_100a.cubin > dis.txt)
"""
import re
import sys
from collections import Counter

path, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur_fn, cur_line = None, None
cnt = Counter()
inside = False
for l in open(path):
    m = re.search(r"\.type\s+\$\S*?\$(\S+),@function", l) or re.search(r"^\s*\.type\s+(\S+),@function", l)
    if m:
        inside = want in m.group(1)
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur_line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if inside and re.search(r"/\*[0-9a-f]{4,}\*/\s", l):
        cnt[cur_line] += 1
tot = sum(cnt.values())
print(f"{tot} instructions ({tot * 16 / 1024:.1f} KB)")
src = {}
for (f, ln), n in cnt.most_common(top):
    if f not in src:
        try:
            src[f] = open(next(p for p in [f"paper_2605_02329_b200/csrc/{f}", f"include/{f}"] if __import__("os").path.exists(p))).read().split("\n")
        except StopIteration:
            src[f] = []
    text = src[f][ln - 1].strip()[:100] if ln - 1 < len(src[f]) else ""
    print(f"{n:5d} {f}:{ln:<5d} {text}")
