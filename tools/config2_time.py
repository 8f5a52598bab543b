"""Device time of config 2 (one 100k-request instance per pair) with the library in SLOSIM_LIB (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config2

sw = config2()
db = DeviceBatch(sw.packed)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
s = db.fetch()
print(f"config2 {e0.elapsed_time(e1):.0f} ms digest {[int(x) for x in s['digest']]}")
