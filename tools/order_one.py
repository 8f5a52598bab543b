"""Run one config5 slice under a named processing order (for ncu metric captures on the GPU box).

usage: python tools/order_one.py ORDER [SLICE]   ORDER in dp,cost | dp,pp,cost | cost
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config5

name = sys.argv[1]
SL = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
sw = config5(select=np.arange(SL, 2 * SL))
inst = sw.packed.instances
fac = inst["rescale_factor"].astype(np.float64)
cost = inst["n_requests"] * np.where(fac > 0, fac, 1.0)
dp = inst["decode_policy"].astype(np.int64)
pp = inst["prefill_policy"].astype(np.int64)
o = {"dp,cost": np.lexsort((-cost, -dp)), "dp,pp,cost": np.lexsort((-cost, -pp, -dp)),
     "cost": np.argsort(-cost, kind="stable")}[name]
db = DeviceBatch(sw.packed, order=o.astype(np.int64))
db.launch(); torch.cuda.synchronize()
db.launch(); torch.cuda.synchronize()
