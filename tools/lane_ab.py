"""Lane engine vs warp engine on config-5 slices (GPU box): timing and field-by-field equality.

usage: python tools/lane_ab.py [SLICE] [STEPS] [variant=ENV=VAL,...]...
Each variant runs in its own process; the first variant is the reference for the equality check.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, time, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import DeviceBatch, config5
SL, STEPS = int(os.environ["AB_SLICE"]), int(os.environ["AB_STEPS"])
sel = np.arange(SL * (STEPS + 1)) % (1 << 20)
sw = config5(select=sel)
db = DeviceBatch(sw.packed)
db.launch_range(0, SL); torch.cuda.synchronize()
ms = []
for k in range(1, STEPS + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); db.launch_range(k * SL, SL); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
h = db.summaries.cpu().numpy().view(_abi.summary_dtype()).copy()
h["sim_cycles"] = 0
np.save(OUT, h)
print(json.dumps({"ms": [round(x, 1) for x in ms], "mreq_s": round(SL * 1000 / (sum(ms) / len(ms)) / 1e3, 2),
                  "status_bad": int((h["status"] != 0).sum())}))
'''
sl = sys.argv[1] if len(sys.argv) > 1 else "16384"
steps = sys.argv[2] if len(sys.argv) > 2 else "3"
variants = sys.argv[3:] or ["warp=SLOSIM_NO_LANE_ENGINE=1", "lane=SLOSIM_X=0"]
import numpy as np

base = None
for v in variants:
    name, rest = v.split("=", 1)
    env = dict(os.environ, AB_SLICE=sl, AB_STEPS=steps)
    for kv in rest.split(","):
        k, val = kv.split("=", 1)
        env[k] = val
    out = f"/tmp/ab_{name}.npy"
    code = CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1800)
    if r.returncode:
        print(name, "FAILED", r.stderr[-2000:])
        continue
    res = json.loads(r.stdout.strip().splitlines()[-1])
    h = np.load(out)
    if base is None:
        base = h
        res["equal"] = "reference"
    else:
        bad = []
        for f in h.dtype.names:
            a, b = h[f], base[f]
            eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
            if not eq:
                idx = np.nonzero(~((a == b) | ((a != a) & (b != b))))[0] if a.dtype.kind == "f" else np.nonzero(a != b)[0]
                bad.append((f, int(len(idx)), int(idx[0])))
        res["equal"] = not bad
        res["mismatch"] = bad[:8]
    print(name, json.dumps(res), flush=True)
