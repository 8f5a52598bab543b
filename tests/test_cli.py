"""The batched CLI vs the reference `slosim` CLI, byte for byte (tests/golden/make_cli_golden.py).

Every scenario is replayed in a fresh directory; exit codes, stdout and the
bytes of every file written (traces, profiles, per-request CSVs, aggregate
JSON, event logs, sweep and merged CSVs) must equal the reference's.
Mirrors the reference tests/test_cli.py cases.
"""

import importlib.util
import os

import pytest

from helpers import GOLDEN, load_golden

_spec = importlib.util.spec_from_file_location("make_cli_golden", os.path.join(GOLDEN, "make_cli_golden.py"))
mcg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(mcg)


@pytest.fixture(scope="module")
def golden():
    return load_golden("cli_golden.json.gz")


def _compare(name, scenarios, golden):
    from paper_2605_02329_b200.cli import main

    got = mcg.run_scenario(main, scenarios[name])
    want = golden[name]
    assert [s["code"] for s in got["steps"]] == [s["code"] for s in want["steps"]]
    assert [s["stdout"] for s in got["steps"]] == [s["stdout"] for s in want["steps"]]
    assert sorted(got["files"]) == sorted(want["files"])
    bad = [f for f in want["files"] if got["files"][f] != want["files"][f]]
    assert not bad, f"{name}: files differ: {bad[:5]}"


@pytest.mark.parametrize("name", sorted(mcg.CPU_SCENARIOS))
def test_cli_cpu_scenarios_match_reference(name, golden):
    _compare(name, mcg.CPU_SCENARIOS, golden)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(mcg.SCENARIOS))
def test_cli_sweeps_match_reference(name, golden):
    _compare(name, mcg.SCENARIOS, golden)


def test_sweep_is_one_launch(monkeypatch):
    """`run` packs every (qps x pair) point into a single slosim_run_batch_host call."""
    from paper_2605_02329_b200 import cli
    from paper_2605_02329_b200.config import ClusterConfig
    from paper_2605_02329_b200.workload import LongTailSpec, gen_longtail

    calls = []

    def fake_run_packed(packed):
        calls.append(len(packed.summaries))
        raise RuntimeError("stop")

    from oracle import oracle
    from paper_2605_02329_b200.pack import BatchBuilder

    monkeypatch.setattr(cli, "run_packed", fake_run_packed)
    monkeypatch.setattr(cli, "BatchBuilder", lambda: BatchBuilder(synth=oracle.synth))
    monkeypatch.setattr(cli, "check_config", lambda cfg, wl: (type("L", (), {"bsz_buckets": [1], "seq_buckets": [1]}), None))
    base = gen_longtail(LongTailSpec(n_requests=20, seed=3))
    with pytest.raises(RuntimeError, match="stop"):
        cli.run_sweep(ClusterConfig(), base, [0.5, 1.0, 2.0],
                      [("fcfs", "continuous"), ("sjf", "kairos-slack"), ("kairos-urgency", "kairos-slack")])
    assert calls == [9]
