"""Device time of every SURVEY Appendix B config (one launch each) + oracle parity on a sample."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02329_b200 import batch as Bt
which = sys.argv[1:] or ["config1", "config3", "config4", "config2"]
for name in which:
    t0 = time.time()
    sw = Bt.CONFIGS[name]()
    tb = time.time() - t0
    db = Bt.DeviceBatch(sw.packed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    db.launch(); torch.cuda.synchronize()
    e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s = db.fetch()
    n = sw.packed.n_requests
    print(f"{name}: {sw.packed.n_instances} instances, {n} requests, build {tb:.1f}s, device {ms:.1f} ms, "
          f"{n/ms*1e3:.3e} req/s, status {np.unique(s['status']).tolist()}, max_active {int(s['max_active'].max())}, "
          f"max_queue {int(s['max_queue'].max())}", flush=True)
