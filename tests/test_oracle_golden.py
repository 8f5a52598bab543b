"""CPU: pin the C oracle (test infrastructure) to golden vectors produced by the reference.

The oracle is the checker for every GPU parity test, so it must itself be
bit-exact against the reference's own outputs (tests/golden/make_golden.py).
"""

import copy
import hashlib
import json

import numpy as np
import pytest

from helpers import (cfg_from_json, load_golden, pack_cases, pack_config1, row_mismatches, summary_mismatches,
                     wl_from_json)
from oracle import oracle
from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.engine import restore_state
from paper_2605_02329_b200.pack import BatchBuilder, trace_words_bound
from paper_2605_02329_b200.workload import trace_arrays_from_requests


@pytest.fixture(scope="module")
def golden():
    return load_golden()


def test_oracle_config1_matches_reference(golden):
    packed, meta = pack_config1(synth=oracle.synth)
    oracle.run_batch(packed, threads=4)
    for i, (qps, pair) in enumerate(meta):
        assert summary_mismatches(packed.summaries[i], golden["config1"][i]["summary"]) == [], (qps, pair)


def test_oracle_reproduces_appendix_c_digests(golden):
    """SHA-256 step digests of SURVEY Appendix C, recomputed from the oracle's event trace."""
    from helpers import pack_config1 as _p

    packed, meta = _p(synth=oracle.synth)
    # rebuild with trace buffers
    from paper_2605_02329_b200.batch import CONFIG1_RATES, PAIRS_2
    from paper_2605_02329_b200.config import ClusterConfig, CostProfile
    from paper_2605_02329_b200.workload import LongTailSpec, longtail_arrays, rescale_factor

    base = longtail_arrays(LongTailSpec())
    bb = BatchBuilder(synth=oracle.synth)
    tid = bb.add_trace(base)
    prof = CostProfile()
    for qps in CONFIG1_RATES:
        for pp, dp in PAIRS_2:
            bb.add_instance(tid, ClusterConfig(prefill_policy=pp, decode_policy=dp, profile=prof),
                            rescale=rescale_factor(base.arrival_us, qps), trace_words=trace_words_bound(base, 8192))
    packed = bb.build(_abi.F_ROWS | _abi.F_EXPORT_LUT)
    oracle.run_batch(packed, threads=4)
    reqs = base.to_requests()
    for i in range(len(meta)):
        rq = copy.deepcopy(reqs)
        events, _, _ = restore_state(rq, base, packed, i, [1], [1])
        h = hashlib.sha256()
        for ev in events:
            if ev["kind"] == "DecodeStepDone":
                h.update(json.dumps([ev["t_us"], sorted(ev["detail"]["batch"]), ev["detail"]["duration_us"]]).encode())
            elif ev["kind"] == "PrefillStepDone":
                h.update(json.dumps([ev["t_us"], ev["detail"]["batch"], ev["detail"]["duration_us"]]).encode())
        assert h.hexdigest()[:16] == golden["config1"][i]["summary"]["digest_c"], meta[i]


def test_oracle_random_cases_match_reference(golden):
    cases = golden["cases"]
    packed, _ = pack_cases(cases, synth=oracle.synth)
    oracle.run_batch(packed, threads=4)
    for i, c in enumerate(cases):
        assert summary_mismatches(packed.summaries[i], c["summary"]) == [], i
        if c["summary"]["status"] == 0:
            assert row_mismatches(packed, i, c["summary"]["rows"]) == [], i


def test_oracle_sparse_profiles_and_bursts_match_reference():
    """File-backed sparse LUTs (general lookup, frozen ground truth) and > 32 active decodes."""
    cases = load_golden("extra_golden.json.gz")
    packed, _ = pack_cases(cases, synth=oracle.synth)
    oracle.run_batch(packed, threads=4)
    for i, c in enumerate(cases):
        assert summary_mismatches(packed.summaries[i], c["summary"]) == [], i
        assert row_mismatches(packed, i, c["summary"]["rows"]) == [], i


def test_oracle_power_of_two_geometry_profiles_match_reference():
    """Fully populated power-of-two LUT grids (file-backed with fractional entries, and synthesized)."""
    cases = load_golden("geo_golden.json.gz")
    packed, _ = pack_cases(cases, synth=oracle.synth)
    oracle.run_batch(packed, threads=4)
    for i, c in enumerate(cases):
        assert summary_mismatches(packed.summaries[i], c["summary"]) == [], i
        if c["summary"]["status"] == 0:
            assert row_mismatches(packed, i, c["summary"]["rows"]) == [], i


def test_oracle_event_logs_match_reference():
    """Full event logs, token timestamps, final LUT and estimator vs Simulation(collect_events=True)."""
    G = load_golden("events_golden.json.gz")
    for k, c in enumerate(G):
        wl = wl_from_json(c["workload"])
        cfg = cfg_from_json(c["config"])
        tr = trace_arrays_from_requests(wl)
        bb = BatchBuilder(synth=oracle.synth)
        bb.add_instance(bb.add_trace(tr), cfg, trace_words=trace_words_bound(tr, cfg.chunk_budget))
        packed = bb.build(_abi.F_ROWS | _abi.F_EXPORT_LUT)
        oracle.run_batch(packed)
        lut = cfg.profile
        bsz = lut.bsz_buckets or [1, 2, 4, 8, 16, 32, 64, 128, 256]
        seq = lut.seq_buckets or [8192 * j for j in range(1, 33)]
        reqs = copy.deepcopy(wl)
        events, lut_out, est = restore_state(reqs, tr, packed, 0, bsz, seq)
        assert events == c["events"], k
        for r in reqs:
            assert r.token_timestamps == c["requests"][r.id]["tokens"], (k, r.id)
            assert r.t_prefill_finish == c["requests"][r.id]["tpf"], (k, r.id)
        assert lut_out._counts.tolist() == c["lut_counts"], k
        assert lut_out._sums.tolist() == [[float(x) for x in row] for row in c["lut_sums"]], k
        assert [est.total_tokens, est.total_busy_us] == c["estimator"], k


def test_oracle_pcg64_matches_numpy():
    """Decode-noise RNG restatement (engine.py:191) vs numpy's own PCG64 stream."""
    from paper_2605_02329_b200.pack import rng_state

    for seed in (0, 5, 123, 2**40 + 7):
        g = np.random.default_rng(seed)
        st = np.array(rng_state(seed), dtype=np.uint64)
        for _ in range(200):
            assert int(oracle.lib().oracle_pcg_next(st.ctypes.data)) == int(g.bit_generator.random_raw())


def test_oracle_policy_snapshots_match_reference():
    P = load_golden("policy_golden.json.gz")
    for c in P["lut"]:
        qb = [q[0] for q in c["queries"]]
        qs = [q[1] for q in c["queries"]]
        got = oracle.lut_lookup(c["bsz"], c["seq"], c["sums"], c["counts"], qb, qs)
        assert got.tolist() == c["values"]
    for c in P["estimate"]:
        toks = np.array(c["tokens"], np.int64)
        out = np.zeros(len(toks), np.int64)
        oracle.lib().oracle_estimate_duration(c["est"][0], c["est"][1], len(toks), toks.ctypes.data, out.ctypes.data)
        assert out.tolist() == c["out"]
