"""Configs 1-4 through the warp engine (default routing) and the lane engine at k live lanes per warp
(SLOSIM_LANE_LPW=k), each in its own process; device ms of the second launch, summaries checked
against the default routing (GPU box).   usage: python tools/lpw_sweep.py [CONFIG ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfgs = sys.argv[1:] or ["config1", "config3", "config4", "config2"]
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import batch as B
sw = B.CONFIGS[CFG]()
db = B.DeviceBatch(sw.packed)
db.launch(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
np.save(OUTF, db.fetch())
print(f"{e0.elapsed_time(e1):.1f}")
'''
import numpy as np

variants = [("default", {})] + [(f"lpw{k}", {"SLOSIM_LANE_LPW": str(k)}) for k in (1, 2, 4, 8, 16, 32)]
for cfg in cfgs:
    ref = None
    for name, env in variants:
        if cfg == "config2" and name in ("lpw4", "lpw8", "lpw16", "lpw32"):
            continue
        outf = f"/tmp/lpw_{cfg}_{name}.npy"
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)).replace("OUTF", repr(outf))
        env2 = dict(os.environ, **env)
        if name == "lpw32":
            env2["SLOSIM_FORCE_LANE_ENGINE"] = "1"
        r = subprocess.run([sys.executable, "-c", code], env=env2, capture_output=True, text=True)
        if r.returncode:
            print(cfg, name, "FAILED", r.stderr[-400:])
            continue
        s = np.load(outf)
        if ref is None:
            ref = s
        bad = [k for k in s.dtype.names if k != "sim_cycles" and not np.array_equal(s[k], ref[k])]
        print(f"{cfg:8s} {name:8s} {float(r.stdout.split()[-1]):9.1f} ms  {'ok' if not bad else 'DIFF ' + str(bad)}",
              flush=True)
