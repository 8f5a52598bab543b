"""GPU probe: launch time vs slice size on config5, and per-instance sim_cycles of one slice.

usage (GPU box): python tools/probe_tail.py  -> gpurun_out/probe_tail.npz + printed table
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_02329_b200 import _abi  # noqa: E402
from paper_2605_02329_b200.batch import DeviceBatch, config5  # noqa: E402

sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "16384", "32768", "65536"])]
n = max(sizes) * 2
t0 = time.time()
sw = config5(select=np.arange(n))
db = DeviceBatch(sw.packed)
print(f"packed {n} instances in {time.time() - t0:.1f}s", flush=True)
db.launch_range(0, 4096)
torch.cuda.synchronize()
res = {}
for sz in sizes:
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        db.launch_range(sz * rep % n, sz)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"slice {sz:6d} rep {rep}: {ms:8.1f} ms  {sz * 1000 / ms / 1e3:6.2f} M req/s", flush=True)
        res[(sz, rep)] = ms
host = db.summaries.cpu().numpy().view(_abi.summary_dtype())
inst = sw.packed.instances
np.savez("gpurun_out/probe_tail.npz", sim_cycles=host["sim_cycles"][:n], dsteps=host["decode_steps"][:n], psteps=host["prefill_steps"][:n], maxact=host["max_active"][:n], v_dec=host["v_dec"][:n],
         b_dec=host["b_dec"][:n], v_pre=host["v_pre"][:n], rescale=inst["rescale_factor"][:n],
         dp=inst["decode_policy"][:n], pp=inst["prefill_policy"][:n], ttft=inst["ttft_slo_us"][:n],
         tpot=inst["tpot_slo_us"][:n], sizes=np.array(sizes), ms=np.array([res[(s, r)] for s in sizes for r in range(2)]))
