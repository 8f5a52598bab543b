"""Build variant libraries for A/B timing: python tools/ab_build.py NAME "-DFOO=1 -DBAR" [NAME2 "..."]

Outputs build/ab/lib_NAME.so (git-ignored; travels with gpurun).
"""
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import _build  # noqa: E402

os.makedirs(os.path.join(ROOT, "build", "ab"), exist_ok=True)
args = sys.argv[1:]
procs = []
for name, flags in zip(args[::2], args[1::2]):
    out = os.path.join(ROOT, "build", "ab", f"lib_{name}.so")
    cmd = [_build.nvcc()] + _build.NVCC_FLAGS + shlex.split(flags) + ["-o", out] + \
        [os.path.join(_build.CSRC, s) for s in _build.SOURCES]
    procs.append((name, out, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
for name, out, p in procs:
    _, err = p.communicate()
    if p.returncode != 0:
        print(f"{name}: FAILED\n{err[-3000:]}")
        continue
    info = [l for l in err.splitlines() if "simulateILi1ELb0" in l or "sim_kernel" in l]
    lines = err.splitlines()
    for i, l in enumerate(lines):
        if "simulateILi1ELb0" in l or ("Function properties for _ZN6slosim10sim_kernel" in l):
            info.append(lines[i + 1].strip())
        if "Compiling entry function '_ZN6slosim10sim_kernel" in l:
            info += [x.strip() for x in lines[i + 2:i + 4]]
    print(f"{name}: ok  " + " | ".join(info[-4:]))
