"""Per-policy-pair share of warp time on one config5 slice (GPU box): sums the engine's per-instance
sim_cycles (clock64 from instance start to finalize) by policy pair, plus cycles per decode step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200.batch import PAIRS_4, DeviceBatch, config5

SL = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sw = config5(select=np.arange(SL, 2 * SL))
db = DeviceBatch(sw.packed)
db.launch(); torch.cuda.synchronize()
db.launch()
s = db.fetch()
cyc = s["sim_cycles"].astype(np.float64)
tot = cyc.sum()
for p, (a, b) in enumerate(PAIRS_4):
    m = sw.coords["pair"] == p
    print(f"{a:>15s}+{b:<12s} share {cyc[m].sum() / tot * 100:5.1f}%  cycles/decode-step "
          f"{cyc[m].sum() / s['decode_steps'][m].sum():7.1f}  cycles/request {cyc[m].sum() / s['n'][m].sum():8.1f}  "
          f"steps/request {s['decode_steps'][m].sum() / s['n'][m].sum():6.1f}")
