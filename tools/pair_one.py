"""One launch of N config-5 instances of one policy pair (profiling target, GPU box).
usage: python tools/pair_one.py N PAIR"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config5

n, p = int(sys.argv[1]), int(sys.argv[2])
idx = np.arange(0, 1 << 20)
idx = idx[idx % 4 == p][:n]
db = DeviceBatch(config5(select=idx).packed)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
print(f"{n} instances of pair {p}: {e0.elapsed_time(e1):.1f} ms")
