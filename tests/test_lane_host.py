"""CPU: the lane engine's per-lane simulation code (csrc/tengine.cuh), compiled as host C++ by the
test harness tools/lane_host (no GPU), against the reference's golden vectors and the C oracle.

The lane engine runs one instance per thread; its decisions must equal the reference's on every
instance it accepts (power-of-two LUT geometry, fully populated LUT, plain ground-truth formula).
The same source is what the CUDA build compiles; tests/test_gpu_lane.py checks the device run.
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from helpers import load_golden, pack_cases, summary_mismatches

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "tools", "lane_host")


@pytest.fixture(scope="module")
def lane():
    subprocess.run(["bash", os.path.join(HARNESS, "build.sh")], check=True)
    L = ctypes.CDLL(os.path.join(HARNESS, "liblane_host.so"))
    L.lane_host_run_batch.argtypes = [ctypes.c_void_p]
    return L


def _run(L, packed):
    b = packed.host_struct()
    L.lane_host_run_batch(ctypes.addressof(b))
    return packed.summaries


@pytest.mark.parametrize("fixture", ["engine_golden.json.gz", "extra_golden.json.gz", "geo_golden.json.gz"])
def test_lane_engine_matches_reference_golden(lane, fixture):
    from oracle import oracle

    g = load_golden(fixture)
    cases = g["cases"] if isinstance(g, dict) else g
    packed, _ = pack_cases(cases, synth=oracle.synth, flags=0)
    got = _run(lane, packed)
    covered = 0
    bad = {}
    for i, c in enumerate(cases):
        if int(got[i]["status"]) == -99:  # outside the lane engine's scope (runs on the warp engine)
            continue
        covered += 1
        m = summary_mismatches(got[i], c["summary"])
        if m:
            bad[i] = m
    assert not bad, f"{len(bad)} of {covered} cases differ: {dict(list(bad.items())[:5])}"
    assert covered > 0


def test_lane_engine_matches_oracle_on_config5_and_config3_samples(lane):
    from oracle import oracle
    from paper_2605_02329_b200 import batch as B

    rng = np.random.default_rng(11)
    for name, sel in [("config5", np.sort(rng.choice(1 << 20, 384, replace=False))),
                      ("config3", np.arange(0, 3072, 13)), ("config4", np.arange(0, 2048, 211))]:
        sw = B.CONFIGS[name](synth=oracle.synth, select=sel)
        ref = B.CONFIGS[name](synth=oracle.synth, select=sel)
        oracle.run_batch(ref.packed, threads=os.cpu_count() or 4)
        got = _run(lane, sw.packed)
        want = ref.packed.summaries
        assert np.all(got["status"] == 0)
        for f in [x for x in want.dtype.names if x != "sim_cycles"]:
            a, b = got[f], want[f]
            eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
            assert eq, (name, f)


def test_lane_engine_matches_oracle_on_random_sweep(lane):
    """The GPU fuzz sweep's random instances (tests/test_gpu_fuzz.py) that the lane engine covers:
    bursts beyond 64 concurrent decodes, KV gating, transfer delays, prefix hits, every policy pair."""
    import importlib.util

    from oracle import oracle

    spec = importlib.util.spec_from_file_location("fuzz", os.path.join(ROOT, "tests", "test_gpu_fuzz.py"))
    fuzz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fuzz)
    packed = fuzz._batch(synth=oracle.synth, n_inst=400)
    got = _run(lane, packed).copy()
    ref = fuzz._batch(synth=oracle.synth, n_inst=400)
    oracle.run_batch(ref, threads=os.cpu_count() or 4)
    want = ref.summaries
    cov = got["status"] != -99
    assert cov.sum() > 100
    assert int(want[cov]["max_active"].max()) > 64
    for f in [x for x in want.dtype.names if x != "sim_cycles"]:
        a, b = got[f][cov], want[f][cov]
        eq = np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)
        assert eq, f
