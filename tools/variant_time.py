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
    bad = [k for k in ref.packed.summaries.dtype.names
           if not np.array_equal(s[sel][k], ref.packed.summaries[k], equal_nan=(s[k].dtype.kind == 'f'))]
    print("parity vs oracle on 512 instances:", "OK" if not bad else bad, flush=True)
