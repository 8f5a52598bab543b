"""Section profile of the engine loop (needs a -DSLOSIM_PROF build, e.g. tools/ab_build.py prof -DSLOSIM_PROF).

usage: SLOSIM_LIB=build/ab/lib_prof.so python tools/prof_sections.py N [PAIR ...]
Prints the share of warp cycles per loop section, by policy pair, for N config5 instances.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import PAIRS_4, DeviceBatch, config5

NAMES = ["rare events", "decode done", "admit+prefill start", "decode start", "fast-forward", "loop top"]
n = int(sys.argv[1])
pairs = [int(x) for x in sys.argv[2:]] or [0, 1, 2, 3]
L = _abi.lib()
L.slosim_prof_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
for p in pairs:
    idx = np.arange(16384, 16384 + 8 * n)
    idx = idx[idx % 4 == p][:n]
    sw = config5(select=idx)
    db = DeviceBatch(sw.packed)
    db.launch(); torch.cuda.synchronize()
    L.slosim_prof_read(buf, 1)
    db.launch(); torch.cuda.synchronize()
    L.slosim_prof_read(buf, 1)
    s = db.fetch()
    v = np.array(buf[:], np.float64)
    steps = s["decode_steps"].sum()
    tot = v[:6].sum()
    print(f"{PAIRS_4[p]}: {tot / 1e9:.1f} Gcycles {tot / steps:.0f} cycles/decode-step, an==1 starts {v[7] / (s['v_dec'].sum() and steps):.2f} "
          f"of steps, ff calls {v[8]:.0f} ff steps {v[9]:.0f} ({v[9] / steps * 100:.1f}% of steps)")
    print(f"   steps with 16 < an <= 32: {(v[6] % 1000000) / steps * 100:.2f}%, an > 32: {(v[6] // 1000000) / steps * 100:.2f}%")
    for k in range(6):
        print(f"   {NAMES[k]:22s} {v[k] / tot * 100:5.1f}%  {v[k] / steps:7.1f} cyc/step")
