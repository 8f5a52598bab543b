"""Generate paper_2605_02329_b200/csrc/rng_tables.h: the constant tables of the workload RNG.

The trace generator of the reference (gen_longtail, /root/reference/pkg/src/slosim/workload.py:88-112)
draws from numpy's Generator (numpy 2.3.5; PCG64, SeedSequence).  The device restatement
(csrc/rng.cuh) needs two sets of constants that are data, not code:

1. numpy's ziggurat tables (numpy/random/src/distributions/ziggurat_constants.h): ki/wi/fi for
   the standard normal, ke/we/fe for the standard exponential, and the tail start points.  They
   are read here out of the installed numpy's compiled ``_generator`` module (the arrays are
   located by their first entries and validated by their defining properties below), so the
   header holds exactly the bits numpy uses.

2. glibc's exp table (__exp_data.tab: 2^(i/128) as scale bits + relative tail, 128 pairs),
   computed here from its definition with exact rational arithmetic and checked against the
   installed libm's copy, which is located the same way.

Run: python tools/gen_rng_tables.py  (rewrites the header; the committed copy is what builds use).
"""

from __future__ import annotations

import glob
import os
import struct
import sys
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2605_02329_b200", "csrc", "rng_tables.h")


def _u64(b, off, n=256):
    return list(struct.unpack_from(f"<{n}Q", b, off))


def _f64(b, off, n=256):
    return list(struct.unpack_from(f"<{n}d", b, off))


def numpy_tables():
    so = glob.glob(os.path.join(os.path.dirname(np.__file__), "random", "_generator*.so"))[0]
    b = open(so, "rb").read()
    ki0, ke0 = struct.pack("<Q", 0x000EF33D8025EF6A), struct.pack("<Q", 0x001C5214272497C6)
    off_ki, off_ke = b.find(ki0), b.find(ke0)
    assert off_ki > 0 and off_ke > 0, "ziggurat tables not found in numpy's _generator module"
    ki = _u64(b, off_ki)
    ke = _u64(b, off_ke)

    # the double arrays: 256 doubles with the defining properties, anywhere in the module
    def find_f64(pred):
        hits = []
        for off in range(0, len(b) - 2048, 8):
            v0 = struct.unpack_from("<d", b, off)[0]
            if not (0 < v0 <= 1.0):
                continue
            a = _f64(b, off)
            if pred(a):
                hits.append((off, a))
        return hits

    def is_f(a):  # fi / fe: f[0] = 1, strictly decreasing, positive
        return a[0] == 1.0 and all(a[i] > a[i + 1] > 0 for i in range(255))

    def is_w(a):  # wi / we: positive widths ~1e-16..1e-15 scale
        return all(0 < x < 1e-12 for x in a)

    fs = find_f64(is_f)
    ws = find_f64(is_w)
    # each kind appears once in _generator: the normal tables are those whose x_i = w_i * 2^52
    # decrease with fi = exp(-x^2/2); the exponential ones satisfy fe = exp(-x)
    def x_of(w, bits):
        return [w[i] * 2.0 ** bits for i in range(256)]

    def pick(cands_w, cands_f, bits, dens):
        for _, w in cands_w:
            xs = x_of(w, bits)
            for _, f in cands_f:
                if all(abs(f[i] - dens(xs[i])) <= 1e-9 for i in range(1, 255)):
                    return w, f
        raise AssertionError("ziggurat table pair not identified")

    wi, fi = pick(ws, fs, 52, lambda x: float(np.exp(-0.5 * x * x)))
    we, fe = pick(ws, fs, 53, lambda x: float(np.exp(-x)))
    # tail starts (ziggurat_constants.h): r and 1/r, located next to each other
    nor_r, exp_r = 3.6541528853610088, 7.69711747013104972
    assert b.find(struct.pack("<d", nor_r)) > 0 and b.find(struct.pack("<d", exp_r)) > 0
    return dict(ki=ki, wi=wi, fi=fi, ke=ke, we=we, fe=fe, nor_r=nor_r, nor_inv_r=0.27366123732975828, exp_r=exp_r)


def _rn(q: Fraction) -> float:
    """Round a positive rational to the nearest double (ties to even)."""
    return float(q)  # Fraction.__float__ is correctly rounded


def _pow2_frac(i: int, n: int, bits: int = 200) -> Fraction:
    """2^(i/n) to `bits` bits (integer n-th root by Newton), as a Fraction."""
    scale = 1 << bits
    target = (1 << i) * scale ** n  # (2^(i/n) * scale)^n = 2^i * scale^n
    x = scale * 2  # upper start
    while True:
        y = ((n - 1) * x + target // x ** (n - 1)) // n
        if y >= x:
            break
        x = y
    return Fraction(x, scale)


def exp_table():
    """__exp_data.tab (EXP_TABLE_BITS = 7): tab[2i] = bits of tail, tab[2i+1] = bits(s) - (i << 45),
    s = RN(2^(i/128)), tail = RN((2^(i/128) - s) / s)."""
    tab = []
    for i in range(128):
        t = _pow2_frac(i, 128)
        s = _rn(t)
        tail = _rn((t - Fraction(s)) / Fraction(s)) if t != Fraction(s) else 0.0
        sb = struct.unpack("<Q", struct.pack("<d", s))[0]
        tab += [struct.unpack("<Q", struct.pack("<d", tail))[0], (sb - (i << 45)) & 0xFFFFFFFFFFFFFFFF]
    return tab


def check_exp_table_against_libm(tab):
    import ctypes.util

    path = None
    for cand in ("/lib/x86_64-linux-gnu/libm.so.6", "/usr/lib/x86_64-linux-gnu/libm.so.6", ctypes.util.find_library("m")):
        if cand and os.path.exists(cand):
            path = cand
            break
    if path is None:
        print("libm not found: exp table unchecked", file=sys.stderr)
        return False
    b = open(path, "rb").read()
    off = b.find(struct.pack("<4Q", *tab[:4]))
    if off < 0:
        # tab[0..1] = (0, 1.0) is too common; search from entry 2
        off = b.find(struct.pack("<4Q", *tab[2:6]))
        off = off - 16 if off >= 0 else off
    ok = off >= 0 and _u64(b, off, 256) == tab
    print(f"exp table vs {path}: {'identical' if ok else 'DIFFERENT'}", file=sys.stderr)
    return ok


def emit(nt, tab):
    def arr(name, ctype, vals, fmt):
        lines = []
        for i in range(0, len(vals), 4):
            lines.append("    " + ", ".join(fmt(v) for v in vals[i:i + 4]) + ",")
        return f"SLOSIM_RNG_TABLE {ctype} {name}[{len(vals)}] = {{\n" + "\n".join(lines) + "\n};\n"

    hexu = lambda v: f"0x{v:016X}ULL"
    hexd = lambda v: f"{float(v).hex()}"
    s = [
        "// rng_tables.h — GENERATED by tools/gen_rng_tables.py; do not edit.",
        "// numpy 2.3.5 ziggurat tables (numpy/random/src/distributions/ziggurat_constants.h, read",
        "// out of the installed numpy's _generator module) and glibc's exp table (__exp_data.tab,",
        "// EXP_TABLE_BITS = 7, computed from its definition and checked against the installed libm).",
        "#pragma once",
        "#include <stdint.h>",
        "#ifndef SLOSIM_RNG_TABLE",
        "#ifdef __CUDACC__",
        "#define SLOSIM_RNG_TABLE static __device__ const",
        "#else",
        "#define SLOSIM_RNG_TABLE static const",
        "#endif",
        "#endif",
        "namespace slosim {",
        "namespace rng {",
        f"constexpr double ZIG_NOR_R = {hexd(nt['nor_r'])};",
        f"constexpr double ZIG_NOR_INV_R = {hexd(nt['nor_inv_r'])};",
        f"constexpr double ZIG_EXP_R = {hexd(nt['exp_r'])};",
        arr("ki_double", "uint64_t", nt["ki"], hexu),
        arr("wi_double", "double", nt["wi"], hexd),
        arr("fi_double", "double", nt["fi"], hexd),
        arr("ke_double", "uint64_t", nt["ke"], hexu),
        arr("we_double", "double", nt["we"], hexd),
        arr("fe_double", "double", nt["fe"], hexd),
        arr("exp_tab", "uint64_t", tab, hexu),
        "}  // namespace rng",
        "}  // namespace slosim",
        "",
    ]
    with open(OUT, "w") as f:
        f.write("\n".join(s))


def main():
    nt = numpy_tables()
    tab = exp_table()
    check_exp_table_against_libm(tab)
    emit(nt, tab)
    print(OUT)


if __name__ == "__main__":
    main()
