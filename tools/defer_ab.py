"""Whole config-5 slice (all four pairs) under environment variants, one process each (GPU box).
usage: python tools/defer_ab.py N name=ENV=VAL[,ENV2=VAL2] ...   ('-' for no env)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200.batch import DeviceBatch, config5
n = NN
sw = config5(select=np.arange(131072, 131072 + 2 * n))
db = DeviceBatch(sw.packed)
db.launch_range(0, n); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch_range(n, n); e1.record(); torch.cuda.synchronize()
s = db.fetch()
print(f"{n * 1000 / e0.elapsed_time(e1) / 1e3:.2f} M req/s digest-xor {int(np.bitwise_xor.reduce(s['digest'][n:2*n])):016x}")
'''
n = int(sys.argv[1])
for v in sys.argv[2:]:
    name, rest = v.split("=", 1)
    env = {} if rest == "-" else dict(kv.split("=", 1) for kv in rest.split(","))
    code = CHILD.replace("ROOT", repr(ROOT)).replace("NN", str(n))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(name, r.stdout.strip() or r.stderr[-400:], flush=True)
