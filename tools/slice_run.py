"""Launch the engine on config5 instances of selected policy pairs (profiling helper, GPU box).

usage: python tools/slice_run.py N [PAIR ...]     (PAIR indexes batch.PAIRS_4; default all)
Runs one warm-up launch and one measured launch of N instances.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config5

n = int(sys.argv[1])
pairs = [int(x) for x in sys.argv[2:]] or [0, 1, 2, 3]
idx = np.arange(16384, 16384 + 8 * n)
idx = idx[np.isin(idx % 4, pairs)][:n]
sw = config5(select=idx)
db = DeviceBatch(sw.packed)
db.launch(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
s = db.fetch()
ms = e0.elapsed_time(e1)
print(f"{n} instances pairs {pairs}: {ms:.1f} ms, {s['n'].sum() / ms * 1e3:.3e} req/s, "
      f"cycles/step {s['sim_cycles'].sum() / s['decode_steps'].sum():.1f}")
