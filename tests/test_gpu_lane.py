"""GPU: the lane engine (csrc/tengine.cuh, one instance per thread) against the oracle and the warp
engine.  The lane engine serves throughput batches; instances outside its scope (general LUT
geometry, frozen ground truth, noise) are deferred to the warp engine in the same launch."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _equal(a, b):
    bad = []
    for f in [x for x in a.dtype.names if x != "sim_cycles"]:
        x, y = a[f], b[f]
        eq = np.array_equal(x, y, equal_nan=True) if x.dtype.kind == "f" else np.array_equal(x, y)
        if not eq:
            bad.append(f)
    return bad


def test_lane_engine_equals_oracle_and_warp_engine_on_config5_sample(monkeypatch):
    import os

    from oracle import oracle
    from paper_2605_02329_b200.batch import config5, run_batch

    rng = np.random.default_rng(2026)
    sel = np.sort(rng.choice(1 << 20, 4096, replace=False))
    monkeypatch.setenv("SLOSIM_FORCE_LANE_ENGINE", "1")
    lane = run_batch(config5(select=sel).packed).copy()
    monkeypatch.delenv("SLOSIM_FORCE_LANE_ENGINE")
    monkeypatch.setenv("SLOSIM_NO_LANE_ENGINE", "1")
    warp = run_batch(config5(select=sel).packed).copy()
    assert _equal(lane, warp) == []
    sub = sel[::8]
    ref = config5(select=sub, synth=oracle.synth)
    oracle.run_batch(ref.packed, threads=os.cpu_count() or 8)
    assert _equal(lane[::8], ref.packed.summaries) == []


def test_mixed_batch_defers_out_of_scope_instances_to_the_warp_engine(monkeypatch):
    """Golden cases of every kind in one launch through the lane path: in-scope instances run on the
    lane engine, file-backed / noisy / non-power-of-two ones are deferred; all match the reference."""
    from helpers import load_golden, pack_cases, summary_mismatches

    from paper_2605_02329_b200.batch import run_batch

    cases = load_golden()["cases"] + load_golden("extra_golden.json.gz") + load_golden("geo_golden.json.gz")
    monkeypatch.setenv("SLOSIM_FORCE_LANE_ENGINE", "1")
    packed, _ = pack_cases(cases, flags=0)
    got = run_batch(packed)
    bad = {i: m for i, c in enumerate(cases) if (m := summary_mismatches(got[i], c["summary"]))}
    assert not bad, f"{len(bad)} cases differ: {dict(list(bad.items())[:5])}"


def test_lane_engine_on_batches_smaller_than_a_warp(monkeypatch):
    """Forced onto a 12-instance batch (config 1), most lanes of the grid never hold an instance:
    they must take part in the cooperative prefill starts without touching any descriptor."""
    from helpers import load_golden, summary_mismatches

    from paper_2605_02329_b200.batch import config1, run_batch

    monkeypatch.setenv("SLOSIM_FORCE_LANE_ENGINE", "1")
    got = run_batch(config1().packed)
    golden = load_golden()["config1"]
    for i in range(12):
        assert summary_mismatches(got[i], golden[i]["summary"]) == [], i
