import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02329_b200.batch import CONFIGS, DeviceBatch
name = sys.argv[1] if len(sys.argv) > 1 else "config3"
kw = {}
if name == "config5":
    kw["select"] = np.arange(0, int(sys.argv[2]) if len(sys.argv) > 2 else 65536)
sw = CONFIGS[name](**kw)
db = DeviceBatch(sw.packed)
db.launch(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    n = sw.packed.n_requests
    print(f"{name}: {sw.packed.n_instances} inst {n} req  {ms:.2f} ms  {n/ms*1e3:.3e} req/s", flush=True)
s = db.fetch()
print("status", np.unique(s["status"]), "e2e", s["e2e_met"][:8])
