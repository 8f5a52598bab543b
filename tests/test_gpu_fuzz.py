"""Randomised GPU-vs-oracle sweep (beyond the reference golden vectors).

Thousands of random instances over every policy pair and knob the engine
specialises on: default and custom bucket grids (the power-of-two geometry path
and the table path), one- to four-anchor decode curves (staged line or general
formula), prefill ground-truth curves, prior weights, noise, transfer delays,
prefix hits, KV limits that gate admission, bursts beyond 32 concurrent decodes (memory mode),
long quiet stretches (fast-forward) and equal arrival times.  Every summary
field and every per-request row must be bit-identical to the C oracle, through
both the throughput and the row-recording specialisations.
"""

import random

import numpy as np
import pytest

from paper_2605_02329_b200.config import ClusterConfig, CostProfile
from paper_2605_02329_b200.domain import Request, SLOConfig
from paper_2605_02329_b200.pack import BatchBuilder
from paper_2605_02329_b200.workload import trace_arrays_from_requests

pytestmark = pytest.mark.gpu

PAIRS = [(p, d) for p in ("fcfs", "sjf", "kairos-urgency") for d in ("continuous", "kairos-slack")]


def _workload(rng, n, k):
    burst = k % 5 == 0
    span = rng.choice([60_000, 2_000_000, 30_000_000, 300_000_000]) if not burst else 50_000
    wl = []
    for i in range(n):
        inp = rng.choice([rng.randrange(1, 3000), rng.randrange(1, 20000), rng.randrange(60000, 140000)])
        inp = rng.randrange(1, 2000) if burst else inp
        wl.append(Request(id=f"f{k}_{i:04d}", arrival_time=rng.randrange(0, span), input_len=inp,
                          output_len=rng.choice([1, rng.randrange(2, 80), rng.randrange(50, 400)]),
                          prefix_hit_len=rng.randrange(0, inp) if rng.random() < 0.1 else 0))
    if rng.random() < 0.15:
        for r in wl[: n // 3]:
            r.arrival_time = span // 2
    wl.sort(key=lambda r: (r.arrival_time, r.id))
    return wl


def _config(rng, wl, k):
    pp, dp = PAIRS[k % len(PAIRS)]
    w = rng.choice([12, 13])
    grid = rng.choice(["default", "default", "pow2", "pow2", "table"])
    bsz = seq = None
    if grid == "pow2":
        bsz = [1 << i for i in range(rng.randrange(2, 10))]
        seq = [(j + 1) << w for j in range(rng.randrange(2, 40))]
    elif grid == "table":
        bsz = sorted(rng.sample(range(1, 300), rng.randrange(2, 9)))
        seq = sorted(rng.sample(range(500, 200_000), rng.randrange(2, 20)))
    anchors = rng.choice([
        [(1, 8192, 11_000), (1, 131072, 40_300)],
        [(1, 16384, 12_500)],
        [(1, 1024, 9_000), (1, 65536, 42_000)],
        [(1, 4096, 7_000), (1, 32768, 15_000), (1, 131072, 60_000), (4, 8192, 30_000)],
    ])
    curve = rng.choice([None, None, [(8192, 400_400), (131072, 8_800_000)], [(5000, 300_000), (50000, 4_000_000)]])
    prof = CostProfile(decode_anchors=anchors, bsz_buckets=bsz, seq_buckets=seq,
                       prior_weight=rng.choice([100, 100, 1, 7]), batch_growth=rng.choice([0.0, 0.03, 0.05]),
                       prefill_gt_curve=curve, decode_noise_eps=rng.choice([0.0, 0.0, 0.0, 0.2]))
    worst = max(r.input_len + r.output_len for r in wl)
    return ClusterConfig(prefill_policy=pp, decode_policy=dp, profile=prof, seed=rng.randrange(1000),
                         kv_capacity_tokens=worst + rng.choice([0, rng.randrange(0, 200_000), 2_000_000]),
                         chunk_budget=rng.choice([2048, 8192]), transfer_base_us=rng.choice([0, 0, 150]),
                         transfer_per_token_us=rng.choice([0.0, 0.0, 0.5]),
                         slo=SLOConfig(ttft_slo_us=rng.choice([8_000_000, 1_000_000]),
                                       tpot_slo_us=rng.choice([50_000, 20_000, 150_000])))


def _batch(synth=None, flags=0, n_inst=1200, seed=20261017):
    rng = random.Random(seed)
    bb = BatchBuilder(synth=synth)
    for k in range(n_inst):
        wl = _workload(rng, rng.randrange(1, 260) if k % 5 else rng.randrange(60, 400), k)
        bb.add_instance(bb.add_trace(trace_arrays_from_requests(wl)), _config(rng, wl, k))
    return bb.build(flags)


@pytest.mark.parametrize("rows", [False, True])
def test_random_instances_equal_oracle(rows):
    from oracle import oracle
    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200.batch import run_batch

    flags = _abi.F_ROWS if rows else 0
    packed = _batch(flags=flags)
    got = run_batch(packed).copy()
    ref = _batch(synth=oracle.synth, flags=flags)
    oracle.run_batch(ref, threads=8)
    want = ref.summaries
    assert np.all(want["status"] == got["status"])
    for k in [x for x in want.dtype.names if x != "sim_cycles"]:
        a, b = got[k], want[k]
        eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
        assert eq, (k, int(np.flatnonzero(a != b)[0]) if not eq and a.dtype.kind != "f" else None)
    if rows:
        for k, v in ref.rows.items():
            assert np.array_equal(packed.rows[k], v, equal_nan=True), k


def test_random_instances_equal_oracle_lane_engine(monkeypatch):
    """The same random sweep forced through the lane engine (one instance per thread); instances outside
    its scope (table grids, partially populated LUTs, noise) are deferred to the warp engine in the same
    launch.  Bursts of up to ~400 requests exercise active sets beyond the 64-entry batch mask."""
    from oracle import oracle
    from paper_2605_02329_b200.batch import run_batch

    monkeypatch.setenv("SLOSIM_FORCE_LANE_ENGINE", "1")
    got = run_batch(_batch()).copy()
    ref = _batch(synth=oracle.synth)
    oracle.run_batch(ref, threads=8)
    want = ref.summaries
    for k in [x for x in want.dtype.names if x != "sim_cycles"]:
        a, b = got[k], want[k]
        eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
        assert eq, (k, int(np.flatnonzero(a != b)[0]) if not eq and a.dtype.kind != "f" else None)


def test_random_instances_equal_oracle_latency_build(monkeypatch):
    """The same random sweep forced through the latency build (one 4-warp block per SM), whose Alg. 3
    runs are fast-forwarded with per-step verification (ff_steps<.., V>): every power-of-two-grid
    kairos-slack instance with more than one request active takes that path whenever a step batches
    the whole active set."""
    from oracle import oracle
    from paper_2605_02329_b200.batch import run_batch

    monkeypatch.setenv("SLOSIM_FORCE_LATENCY_ENGINE", "1")
    got = run_batch(_batch()).copy()
    ref = _batch(synth=oracle.synth)
    oracle.run_batch(ref, threads=8)
    want = ref.summaries
    for k in [x for x in want.dtype.names if x != "sim_cycles"]:
        a, b = got[k], want[k]
        eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
        assert eq, (k, int(np.flatnonzero(a != b)[0]) if not eq and a.dtype.kind != "f" else None)
