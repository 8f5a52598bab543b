"""Cross-check the two GPU engines on all of config 5 (1,048,576 instances), oracle arbitration of
every disagreement (GPU box).  usage: python tools/xcheck.py [N_INSTANCES] [SLICE]

The lane engine and the warp engine are independent implementations of the same semantics; an
instance on which they disagree is re-run on the C oracle (pinned to the reference) to find which
engine is wrong.  Writes gpurun_out/xcheck.json.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
SL = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
CHILD = r'''
import sys, numpy as np, torch, time
sys.path.insert(0, ROOT)
from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import DeviceBatch, config5
sw = config5(select=np.arange(N))
db = DeviceBatch(sw.packed)
t0 = time.time()
for s in range(0, N, SL):
    db.launch_range(s, min(SL, N - s))
torch.cuda.synchronize()
h = db.summaries.cpu().numpy().view(_abi.summary_dtype()).copy()
h["sim_cycles"] = 0
np.save(OUT, h)
print("elapsed", time.time() - t0)
'''
res = {}
for name, env in [("warp", {"SLOSIM_NO_LANE_ENGINE": "1"}), ("lane", {})]:
    out = f"/tmp/xc_{name}.npy"
    code = CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out)).replace("N)", f"{N})").replace("(0, N,", f"(0, {N},").replace("N - s", f"{N} - s").replace("SL", str(SL))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(name, r.stdout.strip(), r.stderr[-500:], flush=True)
    res[name] = np.load(out)
a, b = res["warp"], res["lane"]
diff = np.zeros(len(a), bool)
for f in a.dtype.names:
    x, y = a[f], b[f]
    diff |= ~((x == y) | ((x != x) & (y != y))) if x.dtype.kind == "f" else (x != y)
ids = np.nonzero(diff)[0]
print("instances compared", len(a), "disagreements", len(ids), ids[:20].tolist(), flush=True)
verdict = {}
if len(ids):
    from oracle import oracle
    from paper_2605_02329_b200.batch import config5

    sel = ids[:200]
    ref = config5(select=sel, synth=oracle.synth)
    oracle.run_batch(ref.packed, threads=os.cpu_count() or 8)
    o = ref.packed.summaries.copy()
    o["sim_cycles"] = 0
    for k, ii in enumerate(sel):
        same = lambda h: all((h[ii][f] == o[k][f]) or (h[ii][f] != h[ii][f] and o[k][f] != o[k][f]) for f in o.dtype.names)
        verdict[int(ii)] = {"warp_ok": bool(same(a)), "lane_ok": bool(same(b))}
    print(json.dumps(verdict)[:2000])
json.dump({"n": int(len(a)), "disagreements": ids.tolist(), "verdict": verdict},
          open(os.path.join(ROOT, "gpurun_out", "xcheck.json"), "w"))
