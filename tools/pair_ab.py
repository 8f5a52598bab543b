"""Per policy pair: engine variants on N config-5 instances of one pair (GPU box).
usage: python tools/pair_ab.py N [name=ENV=VAL,ENV2=VAL2 ...]   (default: warp engine vs lane engine)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200.batch import DeviceBatch, config5
n, p = NN, PP
idx = np.arange(0, 1 << 20)
idx = idx[idx % 4 == p][:2 * n]
sw = config5(select=idx)
db = DeviceBatch(sw.packed)
db.launch_range(0, n); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch_range(n, n); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{n * 1000 / ms / 1e3:.2f}")
'''
n = int(sys.argv[1])
variants = []
for v in sys.argv[2:] or ["warp=SLOSIM_NO_LANE_ENGINE=1", "lane=SLOSIM_FORCE_LANE_ENGINE=1"]:
    name, rest = v.split("=", 1)
    variants.append((name, dict(kv.split("=", 1) for kv in rest.split(","))))
for p in range(4):
    out = []
    for name, env in variants:
        code = CHILD.replace("ROOT", repr(ROOT)).replace("NN", str(n)).replace("PP", str(p))
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
        out.append(f"{name} {r.stdout.strip() or r.stderr[-300:]} M req/s")
    print("pair", p, " | ".join(out), flush=True)
