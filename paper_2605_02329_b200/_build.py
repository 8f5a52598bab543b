"""In-tree build of libslosim_b200.so for sm_100a (nvcc, no JIT cache)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libslosim_b200.so")
SOURCES = ["capi.cu", "engine_lat.cu", "longtail.cu"]
HEADERS = ["engine.cuh", "tengine.cuh", "warpops.cuh", "lut.cuh", "numerics.cuh", "rng.cuh", "rng_tables.h", os.path.join("..", "..", "include", "slosim_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "--fmad=false", "-lineinfo",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v",
    "-shared",
]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", OUT + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(r.stderr)
    with open(os.path.join(CSRC, "ptxas_info.txt"), "w") as f:  # register/spill report (no timings: stable diffs)
        f.write("".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l))
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
