"""Shared test helpers: fixture loading and packing (test infrastructure)."""

from __future__ import annotations

import gzip
import json
import math
import os

import numpy as np

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.config import ClusterConfig, CostProfile
from paper_2605_02329_b200.domain import Request, SLOConfig
from paper_2605_02329_b200.pack import BatchBuilder, trace_words_bound
from paper_2605_02329_b200.workload import LongTailSpec, longtail_arrays, rescale_factor, trace_arrays_from_requests

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name="engine_golden.json.gz"):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as f:
        return json.load(f)


_PROFILE_DIR = None


def _profile_file(profile_json) -> str:
    """Materialise a file-backed profile (costmodel.py:312-334 format) for profile_path."""
    global _PROFILE_DIR
    import hashlib
    import tempfile

    if _PROFILE_DIR is None:
        _PROFILE_DIR = tempfile.mkdtemp(prefix="slosim_profiles_")
    text = json.dumps(profile_json, sort_keys=True)
    path = os.path.join(_PROFILE_DIR, hashlib.sha1(text.encode()).hexdigest() + ".json")
    if not os.path.exists(path):
        with open(path, "w") as f:
            f.write(text)
    return path


def cfg_from_json(c) -> ClusterConfig:
    p = c["profile"]
    if p.get("profile_json"):
        prof = CostProfile(profile_path=_profile_file(p["profile_json"]), decode_noise_eps=p["decode_noise_eps"])
        return ClusterConfig(
            chunk_budget=c["chunk_budget"], kv_capacity_tokens=c["kv_capacity_tokens"],
            transfer_base_us=c["transfer_base_us"], transfer_per_token_us=c["transfer_per_token_us"],
            prefill_policy=c["prefill_policy"], decode_policy=c["decode_policy"],
            slo=SLOConfig(c["ttft_slo_us"], c["tpot_slo_us"]), profile=prof, seed=c["seed"],
        )
    prof = CostProfile(
        decode_anchors=[tuple(a) for a in p["decode_anchors"]], batch_growth=p["batch_growth"],
        prior_weight=p["prior_weight"], bsz_buckets=p["bsz_buckets"], seq_buckets=p["seq_buckets"],
        prefill_anchor=tuple(p["prefill_anchor"]),
        prefill_gt_curve=[tuple(x) for x in p["prefill_gt_curve"]] if p["prefill_gt_curve"] else None,
        decode_noise_eps=p["decode_noise_eps"],
    )
    return ClusterConfig(
        chunk_budget=c["chunk_budget"], kv_capacity_tokens=c["kv_capacity_tokens"],
        transfer_base_us=c["transfer_base_us"], transfer_per_token_us=c["transfer_per_token_us"],
        prefill_policy=c["prefill_policy"], decode_policy=c["decode_policy"],
        slo=SLOConfig(c["ttft_slo_us"], c["tpot_slo_us"]), profile=prof, seed=c["seed"],
    )


def wl_from_json(w):
    return [Request(id=a, arrival_time=b, input_len=c, output_len=d, prefix_hit_len=e) for a, b, c, d, e in w]


def pack_cases(cases, synth=None, flags=_abi.F_ROWS, trace=False):
    """One batch holding every golden case as an instance."""
    bb = BatchBuilder(synth=synth)
    traces = []
    for case in cases:
        wl = wl_from_json(case["workload"])
        tr = trace_arrays_from_requests(wl)
        cfg = cfg_from_json(case["config"])
        tid = bb.add_trace(tr)
        bb.add_instance(tid, cfg, trace_words=trace_words_bound(tr, cfg.chunk_budget) if trace else 0)
        traces.append(tr)
    return bb.build(flags), traces


def pack_config1(synth=None, flags=0):
    base = longtail_arrays(LongTailSpec())
    bb = BatchBuilder(synth=synth)
    tid = bb.add_trace(base)
    meta = []
    prof = CostProfile()
    for qps in [0.4, 0.7, 1.0, 1.3, 1.6, 1.9]:
        f = rescale_factor(base.arrival_us, qps)
        for pp, dp in [("fcfs", "continuous"), ("kairos-urgency", "kairos-slack")]:
            bb.add_instance(tid, ClusterConfig(prefill_policy=pp, decode_policy=dp, profile=prof), rescale=f)
            meta.append((qps, f"{pp}+{dp}"))
    return bb.build(flags), meta


SUMMARY_INT_KEYS = ["ttft_met", "tpot_met", "e2e_met", "n_tps", "worst_queue_wait_us", "prefill_steps",
                    "decode_steps", "v_dec", "b_dec", "v_pre", "max_queue", "max_active", "deadline_misses",
                    "est_tokens", "est_busy_us"]


def same_float(a, b):
    if a is None:
        return isinstance(b, float) and math.isnan(b)
    return float(a) == float(b)


def summary_mismatches(got, want):
    """Compare a device/oracle summary row with a golden summary dict; returns list of field names."""
    bad = []
    if want["status"] == 3:
        return [] if int(got["status"]) == 3 else ["status"]
    if int(got["status"]) != 0:
        return ["status"]
    for k in SUMMARY_INT_KEYS:
        if k in want and int(got[k]) != int(want[k]):
            bad.append(k)
    if int(got["digest"]) != int(want["digest"]):
        bad.append("digest")
    for k in ("tps_p50", "tps_p90"):
        if not same_float(want[k], got[k]):
            bad.append(k)
    return bad


def row_mismatches(packed, inst_index, want_rows):
    """Per-request rows of one instance vs golden rows (bit-exact)."""
    R = packed.rows
    off = int(packed.instances[inst_index]["row_offset"])
    bad = []
    for pos_s, w in want_rows.items():
        g = off + int(pos_s)
        checks = [
            ("ttft_us", int(R["ttft_us"][g]) == w["ttft_us"]),
            ("mean_tpot_us", float(R["mean_tpot_us"][g]) == float(w["mean_tpot_us"])),
            ("decode_tps", same_float(w["decode_tps"], R["decode_tps"][g])),
            ("flags", int(R["met_flags"][g]) == w["flags"]),
            ("deadline_misses", int(R["deadline_misses"][g]) == w["deadline_misses"]),
            ("t_prefill_finish", int(R["t_prefill_finish"][g]) == w["t_prefill_finish"]),
            ("t_first_token", int(R["t_first_token"][g]) == w["t_first_token"]),
            ("t_last_token", int(R["t_last_token"][g]) == w["t_last_token"]),
            ("first_sched_us", int(R["first_sched_us"][g]) == w["first_sched_us"]),
        ]
        bad += [(int(pos_s), k) for k, ok in checks if not ok]
    return bad
