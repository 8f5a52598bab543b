"""Config 2 per instance and per engine (GPU box): each policy pair's 100k-request instance launched
alone through the warp engine's latency build and through the lane engine; device ms and ns per
event-loop step, summaries checked equal across engines.
usage: python tools/c2_engines.py [N_REQUESTS]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import batch as B
from paper_2605_02329_b200.workload import LongTailSpec
base, = B._traces([LongTailSpec(n_requests=NREQ, seed=2024, qps=1.0)], "host")
out = []
for k, pair in enumerate(B.PAIRS_2[::-1]):
    sw = B.grid_batch([base], None, [1.0], [pair], name="c2")
    db = B.DeviceBatch(sw.packed)
    db.launch(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
    s = db.fetch()
    ms = e0.elapsed_time(e1)
    steps = int(s["decode_steps"][0] + s["prefill_steps"][0])
    print(f"  {ENGINE:9s} {str(pair):40s} {ms:9.1f} ms  {1e6 * ms / steps:7.1f} ns/step  digest {int(s['digest'][0])}")
    out.append(s)
np.save(OUTF, np.concatenate(out))
'''
res = {}
for name, env in [("warp_lat", {"SLOSIM_FORCE_LATENCY_ENGINE": "1"}), ("lane", {"SLOSIM_FORCE_LANE_ENGINE": "1"}),
                  ("lane_solo", {"SLOSIM_LANE_LPW": "1"})]:
    outf = f"/tmp/c2_{name}.npy"
    code = (CHILD.replace("ROOT", repr(ROOT)).replace("NREQ", str(n_req)).replace("OUTF", repr(outf))
            .replace("ENGINE", repr(name)))
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), check=True)
    import numpy as np
    res[name] = np.load(outf)
a = res["warp_lat"]
for name, b in res.items():
    bad = [k for k in a.dtype.names if k != "sim_cycles" and not np.array_equal(a[k], b[k])]
    print(f"{name}: " + ("agrees with warp_lat" if not bad else f"DIFFERS on {bad}"))
