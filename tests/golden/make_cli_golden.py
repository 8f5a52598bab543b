"""Generate CLI golden fixtures by running the REFERENCE `slosim` CLI (cli.py main()).

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Each scenario writes its input files into an empty directory, then runs a
list of CLI invocations there (relative paths, so the files it writes do not
depend on where it ran) and records every invocation's exit code and stdout,
plus the bytes of every file the scenario directory holds at the end.
tests/test_cli.py replays the same scenarios through paper_2605_02329_b200.cli
and compares bytes.
"""

from __future__ import annotations

import contextlib
import gzip
import io
import json
import os
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

BASE_CLUSTER = {
    "chunk_budget": 8192,
    "kv_capacity_tokens": 500_000,
    "profile": {"decode_anchors": [[1, 8192, 11000], [1, 131072, 40300]], "prefill_anchor": [131072, 8_800_000]},
    "seed": 7,
}


def _cfg(**kw):
    c = {"cluster": BASE_CLUSTER, "workload": {"trace": "trace.jsonl"}, "qps_sweep": [2.0, 3.0],
         "policies": [["fcfs", "continuous"], ["kairos-urgency", "kairos-slack"]], "output_dir": "out"}
    c.update(kw)
    return json.dumps(c, indent=1)


SCENARIOS = {
    # reference tests/test_cli.py base_config + write_small_trace, with event logs
    "sweep_events": {
        "inputs": {"config.json": _cfg()},
        "steps": [["gen-trace", "--out", "trace.jsonl", "--n", "40", "--qps", "2.0", "--seed", "5"],
                  ["run", "--config", "config.json", "--events"]],
    },
    # file-backed profile from profile-synth, decode noise, three policy pairs, --seed override
    "noise_profile_file": {
        "inputs": {"config.json": _cfg(
            cluster={"chunk_budget": 4096, "kv_capacity_tokens": 900_000, "transfer_base_us": 2000,
                     "transfer_per_token_us": 0.05, "slo": {"ttft_slo_us": 3_000_000, "tpot_slo_us": 60_000},
                     "profile": {"profile_path": "profile.json", "decode_noise_eps": 0.2}, "seed": 3},
            qps_sweep=[1.0, 2.5],
            policies=[["sjf", "kairos-slack"], ["kairos-urgency", "continuous"], ["fcfs", "kairos-slack"]])},
        "steps": [["gen-trace", "--out", "trace.jsonl", "--n", "60", "--qps", "1.5", "--seed", "9", "--p-long", "0.2",
                   "--long-min", "20000", "--long-max", "60000"],
                  ["profile-synth", "--anchor", "1:8192:11000", "--anchor", "1:131072:40300", "--anchor",
                   "8:65536:30000", "--gamma", "0.05", "--prefill-tokens", "65536", "--prefill-duration-us",
                   "4000000", "--out", "profile.json"],
                  ["run", "--config", "config.json", "--seed", "99", "--events"]],
    },
    # generated long-tail workload, piecewise ground-truth prefill curve, custom buckets
    "longtail_curve": {
        "inputs": {"config.json": json.dumps({
            "cluster": {"chunk_budget": 2048, "kv_capacity_tokens": 400_000,
                        "profile": {"decode_anchors": [[1, 4096, 9000], [4, 65536, 30000]], "batch_growth": 0.02,
                                    "bsz_buckets": [1, 2, 4, 8, 16, 32], "seq_buckets": [4096 * k for k in range(1, 17)],
                                    "prefill_anchor": [16384, 1_500_000],
                                    "prefill_gt_curve": [[1024, 120000], [8192, 700000], [16384, 1500000]]}},
            "workload": {"longtail": {"n_requests": 150, "qps": 1.0, "seed": 4, "p_long": 0.1,
                                      "long_len_min": 20000, "long_len_max": 60000}},
            "qps_sweep": [0.7, 1.3],
            "policies": [["fcfs", "continuous"], ["kairos-urgency", "kairos-slack"]],
            "output_dir": "lt"})},
        "steps": [["run", "--config", "config.json"]],
    },
    # sweeps merged by `report` (reference test_report_merges_sweeps)
    "report_merge": {
        "inputs": {"c1.json": _cfg(qps_sweep=[3.0], output_dir="s1"), "c2.json": _cfg(qps_sweep=[2.0], output_dir="s2")},
        "steps": [["gen-trace", "--out", "trace.jsonl", "--n", "40", "--qps", "2.0", "--seed", "5"],
                  ["run", "--config", "c1.json"], ["run", "--config", "c2.json"],
                  ["report", "s1/sweep.csv", "s2/sweep.csv", "--out", "merged.csv"]],
    },
    # a request that never fits KV: exit 3 before any output (test_run_impossible_capacity_exits_3)
    "capacity_exit3": {
        "inputs": {"config.json": _cfg(cluster=dict(BASE_CLUSTER, kv_capacity_tokens=10))},
        "steps": [["gen-trace", "--out", "trace.jsonl", "--n", "40", "--qps", "2.0", "--seed", "5"],
                  ["run", "--config", "config.json"]],
    },
}

# scenarios whose steps run without a GPU in the replay (gen-trace, argument/config errors)
CPU_SCENARIOS = {
    "gen_trace_only": {
        "inputs": {},
        "steps": [["gen-trace", "--out", "a.jsonl", "--n", "30", "--seed", "11"],
                  ["gen-trace", "--out", "b.jsonl", "--n", "80", "--qps", "3.5", "--seed", "2", "--p-long", "0.3",
                   "--long-min", "1000", "--long-max", "5000", "--short-log-mean", "6.0", "--out-log-sigma", "1.1"]],
    },
    "config_errors": {
        "inputs": {"ambiguous.json": _cfg(workload={"trace": "trace.jsonl", "longtail": {"n_requests": 5}}),
                   "unknown_key.json": _cfg(cluster=dict(BASE_CLUSTER, mystery_knob=1)),
                   "missing_trace.json": _cfg(workload={"trace": "nope.jsonl"}),
                   "no_policies.json": _cfg(policies=[]),
                   "bad_qps.json": _cfg(qps_sweep=[1.0, -2.0])},
        "steps": [["gen-trace", "--out", "trace.jsonl", "--n", "10", "--seed", "5"],
                  ["run", "--config", "ambiguous.json"], ["run", "--config", "unknown_key.json"],
                  ["run", "--config", "missing_trace.json"], ["run", "--config", "no_policies.json"],
                  ["run", "--config", "bad_qps.json"], ["report", "missing.csv", "--out", "m.csv"]],
    },
}


def run_scenario(main, sc) -> dict:
    """Replay one scenario with the CLI `main` in a fresh directory; return its record."""
    old = os.getcwd()
    with tempfile.TemporaryDirectory() as d:
        os.chdir(d)
        try:
            for name, text in sc["inputs"].items():
                with open(name, "w", encoding="utf-8") as f:
                    f.write(text)
            steps = []
            for argv in sc["steps"]:
                out = io.StringIO()
                with contextlib.redirect_stdout(out), contextlib.redirect_stderr(io.StringIO()):
                    code = main(list(argv))
                steps.append({"argv": argv, "code": code, "stdout": out.getvalue()})
            files = {}
            for root, _, names in os.walk("."):
                for n in names:
                    p = os.path.normpath(os.path.join(root, n))
                    with open(p, encoding="utf-8") as f:
                        files[p] = f.read()
            return {"steps": steps, "files": dict(sorted(files.items()))}
        finally:
            os.chdir(old)


def main() -> None:
    sys.path.insert(0, REF)
    from slosim.cli import main as ref_main

    out = {}
    for name, sc in {**SCENARIOS, **CPU_SCENARIOS}.items():
        rec = run_scenario(ref_main, sc)
        out[name] = rec
        print(name, [s["code"] for s in rec["steps"]], len(rec["files"]), "files")
    with gzip.open(os.path.join(HERE, "cli_golden.json.gz"), "wt", encoding="utf-8") as f:
        json.dump(out, f, sort_keys=True)


if __name__ == "__main__":
    main()
