"""One config-2-style instance (100k-request trace seed 2024 qps 1.0, truncated to N requests) of one
policy pair, launched once (ncu target, GPU box).  usage: python tools/c2_one.py N PAIR_INDEX"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_02329_b200 import batch as B
from paper_2605_02329_b200.workload import LongTailSpec

n, k = int(sys.argv[1]), int(sys.argv[2])
base, = B._traces([LongTailSpec(n_requests=n, seed=2024, qps=1.0)], "host")
pair = B.PAIRS_2[::-1][k]
db = B.DeviceBatch(B.grid_batch([base], None, [1.0], [pair], name="c2one").packed)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
s = db.fetch()
steps = int(s["decode_steps"][0] + s["prefill_steps"][0])
print(f"{pair} n={n}: {e0.elapsed_time(e1):.1f} ms, {1e6 * e0.elapsed_time(e1) / steps:.1f} ns/step")
