"""Run chosen config-5 instances alone on the GPU through each engine and the oracle; print the
fields that differ (GPU box debugging aid).

usage: python tools/one_instance.py ID [ID ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

ids = np.array([int(x) for x in sys.argv[1:]], np.int64)
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ROOT)
from paper_2605_02329_b200.batch import config5, run_batch
ids = np.array(IDS, np.int64)
got = run_batch(config5(select=ids).packed)
np.save(OUT, got)
'''
res = {}
for name, env in [("warp_lat", {"SLOSIM_FORCE_LATENCY_ENGINE": "1"}), ("warp_thr", {"SLOSIM_NO_LATENCY_ENGINE": "1", "SLOSIM_NO_LANE_ENGINE": "1"}),
                  ("lane", {"SLOSIM_FORCE_LANE_ENGINE": "1"})]:
    out = f"/tmp/one_{name}.npy"
    code = CHILD.replace("ROOT", repr(ROOT)).replace("IDS", repr(ids.tolist())).replace("OUT", repr(out))
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), check=True)
    res[name] = np.load(out)
from oracle import oracle
from paper_2605_02329_b200.batch import config5

ref = config5(select=ids, synth=oracle.synth)
oracle.run_batch(ref.packed, threads=4)
res["oracle"] = ref.packed.summaries
for i, ii in enumerate(ids):
    print("instance", ii)
    for f in ["status", "ttft_met", "tpot_met", "e2e_met", "decode_steps", "prefill_steps", "v_dec", "b_dec", "digest",
              "tps_p50", "deadline_misses", "max_active"]:
        vals = {k: v[i][f].item() for k, v in res.items()}
        flag = "" if len(set(str(x) for x in vals.values())) == 1 else "   <-- differs"
        print(f"  {f:16s} {vals}{flag}")
