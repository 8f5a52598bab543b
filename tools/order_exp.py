"""Work-order experiment (GPU box): time one config5 slice under different processing orders.

usage: python tools/order_exp.py [SLICE]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import DeviceBatch, config5

SL = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sw = config5(select=np.arange(SL, 2 * SL))
inst = sw.packed.instances
fac = inst["rescale_factor"].astype(np.float64)
cost = inst["n_requests"] * np.where(fac > 0, fac, 1.0)
dp = inst["decode_policy"].astype(np.int64)
pp = inst["prefill_policy"].astype(np.int64)
orders = {
    "dp,cost": np.lexsort((-cost, -dp)),
    "dp,pp,cost": np.lexsort((-cost, -pp, -dp)),
    "cost": np.argsort(-cost, kind="stable"),
    "pp,dp,cost": np.lexsort((-cost, -dp, -pp)),
}
for name, o in orders.items():
    db = DeviceBatch(sw.packed, order=o.astype(np.int64))
    db.launch(); torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"{name:12s} {min(ms):8.1f} ms  {SL * 1000 / min(ms) * 1e3 / 1e6:6.2f} M req/s", flush=True)
