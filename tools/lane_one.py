"""One config-5 launch of N instances through the lane engine (profiling target, GPU box).
usage: python tools/lane_one.py N [START]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config5

n = int(sys.argv[1])
start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sw = config5(select=np.arange(start, start + n) % (1 << 20))
db = DeviceBatch(sw.packed)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
s = db.fetch()
ms = e0.elapsed_time(e1)
print(f"{n} instances: {ms:.1f} ms, {s['n'].sum() / ms * 1e3:.3e} req/s, bad status {(s['status'] != 0).sum()}")
