"""Run ALL of config 5 (1,048,576 instances, 1.05e9 simulated requests) on one GPU in 16,384-instance
launches, build the per-(pair, rate, SLO) e2e-attainment histograms, and check a random sample of
instances against the C oracle.  Writes gpurun_out/full_sweep.json.

usage (GPU box): python tools/full_sweep.py [SAMPLE]
"""
import ctypes
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200 import dist as D
from paper_2605_02329_b200.batch import DeviceBatch, config5

SL = 16384
sample = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
t0 = time.time()
sw = config5()
db = DeviceBatch(sw.packed)
n = sw.packed.n_instances
build_s = time.time() - t0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for s in range(0, n, SL):
    db.launch_range(s, SL)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
summ = db.summaries.cpu().numpy().view(_abi.summary_dtype())
assert np.all(summ["status"] == 0)
cells = D.cell_ids_config_grid(np.arange(n), 4, 16, 64)
hist = np.zeros((4 * 16 * 64, 1001), np.int64)
np.add.at(hist, (cells, summ["e2e_met"]), 1)
# oracle check on a random sample
from oracle import oracle

sel = np.sort(np.random.default_rng(7).choice(n, sample, replace=False))
ref = config5(select=sel, synth=oracle.synth)
t1 = time.time()
oracle.run_batch(ref.packed, threads=os.cpu_count() or 1)
cpu_s = time.time() - t1
bad = [k for k in ref.packed.summaries.dtype.names if k != "sim_cycles" and
       not np.array_equal(summ[sel][k], ref.packed.summaries[k], equal_nan=True)]
reqs = int(summ["n"].astype(np.int64).sum())
out = {"instances": int(n), "requests": reqs, "device_s": ms / 1e3, "req_per_s": reqs / (ms / 1e3),
       "launches": (n + SL - 1) // SL, "host_build_s": build_s,
       "hist_sha256": hashlib.sha256(hist.tobytes()).hexdigest()[:16],
       "oracle_sample": int(sample), "oracle_sample_s": cpu_s, "oracle_threads": os.cpu_count(),
       "mismatched_fields": bad, "e2e_attainment_mean": float(summ["e2e_met"].sum() / reqs)}
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/full_sweep.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
