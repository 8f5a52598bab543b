"""Time variant libraries on config5 slices (GPU box): python tools/ab_time.py base:lib_base.so v1:lib_v1.so ...

Each variant runs in its own process (SLOSIM_LIB), 1 warm-up + 3 timed 16384-instance slices; summaries of
every variant are compared field-by-field with the first one (exactness guard; sim_cycles excluded).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import DeviceBatch, config5
SL = int(os.environ.get("AB_SLICE", "16384")); STEPS = int(os.environ.get("AB_STEPS", "3"))
sel = np.arange(SL * (STEPS + 1))
sw = config5(select=sel)
db = DeviceBatch(sw.packed)
db.launch_range(0, SL); torch.cuda.synchronize()
ms = []
for k in range(1, STEPS + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); db.launch_range(k * SL, SL); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
h = db.summaries.cpu().numpy().view(_abi.summary_dtype())
np.save(OUT, h)
cyc = h["sim_cycles"].astype(np.float64)
pair = np.arange(len(h)) % 4
by = [float(cyc[(pair == p) & (np.arange(len(h)) >= STEPS * SL)].sum()) for p in range(4)]
print(json.dumps({"ms": ms, "mreq_s": SL * 1000 / (sum(ms) / len(ms)) / 1e3, "gcyc_by_pair_last": [round(x / 1e9, 2) for x in by]}))
'''

res = {}
base = None
for spec in sys.argv[1:]:
    name, lib = spec.split(":")
    lib = lib if os.path.isabs(lib) else os.path.join(ROOT, "build", "ab", lib)
    out = f"/tmp/ab_{name}.npy"
    env = dict(os.environ, SLOSIM_LIB=lib)
    code = CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if p.returncode != 0:
        print(name, "FAILED", p.stderr[-2000:])
        continue
    r = json.loads(p.stdout.strip().splitlines()[-1])
    import numpy as np
    h = np.load(out)
    if base is None:
        base = h
        r["exact"] = True
    else:
        bad = [k for k in h.dtype.names if k != "sim_cycles" and not np.array_equal(h[k], base[k], equal_nan=True)]
        r["exact"] = not bad
        if bad:
            r["mismatch"] = bad
    res[name] = r
    print(f"{name:14s} {r['mreq_s']:7.3f} M req/s  ms={['%.1f' % x for x in r['ms']]}  exact={r['exact']}  "
          f"warp Gcycles by pair (last slice) {r['gcyc_by_pair_last']}", flush=True)
