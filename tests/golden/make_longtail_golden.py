"""Golden traces of the REFERENCE generator gen_longtail (workload.py:88-112), for the device
trace generator.  Run in the build container (where /root/reference exists):

    python tests/golden/make_longtail_golden.py

Imports /root/reference/pkg/src/slosim unmodified and records, per spec, the trace as
(id, arrival_time, input_len, output_len, prefix_hit_len) in the reference's list order:
in full for the small specs, as a SHA-256 of the packed int64 columns for the rest
(configs 2, 4 and all 256 config-5 seeds).  The GPU box never needs /root/reference.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def spec_dict(s):
    return {k: getattr(s, k) for k in ("qps", "n_requests", "short_len_log_mean", "short_len_log_sigma", "p_long",
                                       "long_len_min", "long_len_max", "out_len_log_mean", "out_len_log_sigma",
                                       "seed")}


def trace_sha(reqs) -> str:
    cols = np.array([[r.arrival_time, r.input_len, r.output_len, r.prefix_hit_len] for r in reqs], np.int64)
    return hashlib.sha256(cols.reshape(-1, 4).tobytes()).hexdigest()


def main():
    sys.path.insert(0, REF)
    import slosim

    S = slosim.LongTailSpec
    full = [S(), S(n_requests=1, seed=5), S(n_requests=500, p_long=1.0, seed=6),
            S(n_requests=500, short_len_log_sigma=0.0, out_len_log_sigma=0.0, seed=8),
            S(n_requests=2000, qps=250.0, seed=2**40 + 3), S(n_requests=300, long_len_min=1, long_len_max=2**31 - 2,
                                                             p_long=0.3, seed=12)]
    hashed = ([S(n_requests=100_000, seed=2024, qps=1.0)] + [S(n_requests=20_000, seed=s, qps=4.0) for s in range(8)]
              + [S(seed=s) for s in range(256)])
    out = {"meta": {"numpy": np.__version__, "reference": "slosim @ " + REF}, "full": [], "sha256": []}
    for s in full:
        reqs = slosim.gen_longtail(s)
        out["full"].append({"spec": spec_dict(s), "ids": [r.id for r in reqs],
                            "rows": [[r.arrival_time, r.input_len, r.output_len, r.prefix_hit_len] for r in reqs]})
    for s in hashed:
        reqs = slosim.gen_longtail(s)
        ids_in_order = all(r.id == f"r{k:0{max(4, len(str(max(s.n_requests, 1))))}d}" for k, r in enumerate(reqs))
        out["sha256"].append({"spec": spec_dict(s), "sha256": trace_sha(reqs), "ids_in_position_order": ids_in_order})
    with gzip.open(os.path.join(HERE, "longtail_golden.json.gz"), "wt", encoding="utf-8") as f:
        json.dump(out, f)
    print("wrote", len(out["full"]), "full and", len(out["sha256"]), "hashed traces")


if __name__ == "__main__":
    main()
