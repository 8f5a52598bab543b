"""First differing decode/prefill event between the GPU warp engine (traced) and the oracle for one
config-5 instance; also the untraced GPU summary (GPU box debugging aid).

usage: python tools/trace_diff.py ID
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle import oracle
from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import config5, run_batch
from paper_2605_02329_b200.engine import decode_trace, run_packed

ii = int(sys.argv[1])
WORDS = 30_000_000


def traced(synth):
    sw = config5(select=np.array([ii]), synth=synth)
    pk = sw.packed
    pk.flags = _abi.F_ROWS
    from paper_2605_02329_b200.pack import PackedBatch
    pk2 = PackedBatch(pk.arrival, pk.inp, pk.out, pk.hit, pk.idr, pk.profiles, pk.instances.copy(), _abi.F_ROWS,
                      int(pk.instances["n_requests"].sum()), WORDS)
    pk2.instances["trace_buf_offset"] = 0
    pk2.instances["trace_buf_words"] = WORDS
    return pk2


g = traced(None)
run_packed(g)
o = traced(oracle.synth)
oracle.run_batch(o, threads=1)
try:
    eg = [r for r in decode_trace(g.trace_buf) if r[0] in (2, 3)]
except Exception as ex:
    print("gpu trace:", ex)
    import re
    k = int(re.search(r"word (\d+)", str(ex)).group(1))
    w = g.trace_buf
    # walk records up to k, print the last few
    recs, j = [], 0
    while j < k:
        kind = int(w[j]); start = j
        if kind in (0, 1): j += 3
        elif kind == 4: j += 4
        elif kind == 2: j += 4 + int(w[j + 3])
        elif kind == 3: j += 5 + int(w[j + 3])
        else: break
        recs.append((start, w[start:j].tolist()))
    # active-set size along the run (admits of out>1 requests minus retirements), last records
    outl = {int(p): int(x) for p, x in enumerate(g.out[:1000])}
    act, ngen = set(), {}
    for st, r in recs:
        if r[0] == 4 and outl[r[2]] > 1:
            act.add(r[2]); ngen[r[2]] = 0
        elif r[0] == 3:
            for m in r[5:5 + r[3]]:
                ngen[m] += 1
                if ngen[m] == outl[m] - 1:
                    act.discard(m)
        r.append(("an", len(act)))
    for st, r in recs[-14:]:
        print("  @", st, r[:8], "...", r[-1])
    print("  words at", k, w[k - 2:k + 12].tolist())
    eo = [r for r in decode_trace(o.trace_buf) if r[0] in (2, 3)]
    sys.exit(0)
eo = [r for r in decode_trace(o.trace_buf) if r[0] in (2, 3)]
print("traced gpu summary", g.summaries[0][["decode_steps", "digest", "tpot_met"]], "oracle", o.summaries[0][["decode_steps", "digest", "tpot_met"]])
plain = run_batch(config5(select=np.array([ii])).packed)
print("untraced gpu summary", plain[0][["decode_steps", "digest", "tpot_met"]])
norm = lambda r: (r[0], r[1], r[2], r[3], r[4], tuple(sorted(r[5]))) if r[0] == 3 else (r[0], r[1], r[2], tuple(r[3]))
for k, (a, b) in enumerate(zip(eg, eo)):
    if norm(a) != norm(b):
        print("first difference at event", k)
        for x in range(max(0, k - 3), k + 2):
            print("  gpu", str(eg[x])[:200])
            print("  ora", str(eo[x])[:200])
        break
else:
    print("traced event streams equal over", min(len(eg), len(eo)), "events")
