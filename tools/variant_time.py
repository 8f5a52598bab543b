"""Time config5 slices with a given library variant (SLOSIM_LIB) and check parity vs the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02329_b200.batch import config5, DeviceBatch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sw = config5(select=np.arange(n))
db = DeviceBatch(sw.packed)
db.launch(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for rep in range(2):
    e0.record(); db.launch(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
s = db.fetch().copy()
ms = min(ts)
print(f"{os.environ.get('SLOSIM_LIB','default')}: {n} inst {ms:.1f} ms {sw.packed.n_requests/ms*1e3:.3e} req/s", flush=True)
if len(sys.argv) > 2:
    from oracle import oracle
    sel = np.random.default_rng(0).choice(n, 512, replace=False)
    ref = config5(select=sel, synth=oracle.synth)
    oracle.run_batch(ref.packed, threads=os.cpu_count())
    bad = [k for k in ref.packed.summaries.dtype.names if k != 'sim_cycles'
           if not np.array_equal(s[sel][k], ref.packed.summaries[k], equal_nan=(s[k].dtype.kind == 'f'))]
    print("parity vs oracle on 512 instances:", "OK" if not bad else bad, flush=True)
cyc = s["sim_cycles"].astype(np.float64)
dp = sw.packed.instances["decode_policy"]
print(f"  sim_cycles mean {cyc.mean():.3e} max {cyc.max():.3e} p99 {np.percentile(cyc,99):.3e}; "
      f"kairos-decode mean {cyc[dp==1].mean():.3e} continuous mean {cyc[dp==0].mean():.3e}; "
      f"sum/elapsed-equivalent warps {cyc.sum()/(ms*1e-3*1.965e9):.0f}")
import collections
rates = sw.coords["rate"]
for q in (0.1, 0.5, 1.0, 2.0, 3.25):
    m = np.isclose(rates, q)
    if m.any(): print(f"  rate {q}: mean cycles {cyc[m].mean():.3e}")
