"""GPU: the drop-in API (paper_2605_02329_b200 mirrors slosim) against reference outputs.

* Simulation(collect_events=True): event logs, token timestamps, final LUT and
  estimator vs the reference's own (events_golden.json.gz);
* policy snapshots (LUT lookup, decode/prefill selection, estimator, synth)
  vs reference outputs (policy_golden.json.gz);
* the known-answer behaviours the reference's test suite pins,
  restated as fresh tests against this package.
"""


import numpy as np
import pytest

from helpers import cfg_from_json, load_golden, wl_from_json

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2605_02329_b200")


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_2605_02329_b200 import _abi

    return _abi.lib()


# ------------------------------------------------------------ golden logs --
def test_simulation_event_logs_match_reference():
    G = load_golden("events_golden.json.gz")
    for k, c in enumerate(G):
        wl = wl_from_json(c["workload"])
        sim = S.Simulation(cfg_from_json(c["config"]), wl, collect_events=True)
        sim.run()
        assert sim.events == c["events"], k
        for r in sim.requests:
            assert r.token_timestamps == c["requests"][r.id]["tokens"], (k, r.id)
            assert r.t_prefill_finish == c["requests"][r.id]["tpf"]
            assert r.phase == S.Phase.FINISHED
        assert sim.lut._counts.tolist() == c["lut_counts"], k
        assert [sim.estimator.total_tokens, sim.estimator.total_busy_us] == c["estimator"]
        assert all(r.token_timestamps == [] for r in wl)  # caller's workload untouched


def test_policy_snapshots_match_reference():
    P = load_golden("policy_golden.json.gz")
    for c in P["lut"]:
        lut = S.DecodeStepLUT(c["bsz"], c["seq"])
        lut._sums[:, :] = np.array(c["sums"], np.float64)
        lut._counts[:, :] = np.array(c["counts"])
        got = lut.lookup_many([q[0] for q in c["queries"]], [q[1] for q in c["queries"]])
        assert got.tolist() == c["values"]
    for c in P["decode"]:
        lut = S.DecodeStepLUT(c["bsz"], c["seq"])
        lut._sums[:, :] = np.array(c["sums"], np.float64)
        lut._counts[:, :] = np.array(c["counts"])
        active = []
        for rid, inp, ngen, tf in c["active"]:
            r = S.Request(id=rid, arrival_time=0, input_len=inp, output_len=200)
            r.record_first_token(tf)
            for j in range(ngen):
                r.record_decode_token(j + 1)
            active.append(r)
        sel = S.DECODE_POLICIES[c["policy"]](active, c["t_now"], S.SLOConfig(), lut)
        assert sel.batch == c["batch"] and sel.delayed == c["delayed"]
        assert sel.predicted_step_time_us == c["pred"] and sel.fallback == c["fallback"]
        assert sel.admission_step_times_us == c["times"]
        if c["smin"] is not None:
            assert sel.s_min_us == c["smin"]
    for c in P["prefill"]:
        q = [S.Request(id=a, arrival_time=b, input_len=i, output_len=1, prefix_hit_len=h, prefill_done_tokens=d)
             for a, b, i, h, d in c["queue"]]
        est = S.PrefillThroughputEstimator(*c["est"])
        b = S.PREFILL_POLICIES[c["policy"]](q, c["budget"], c["t_now"], est, S.SLOConfig())
        assert [list(e) for e in b.entries] == c["entries"]
        if c["finishes"] is not None:
            from paper_2605_02329_b200.prefill_sched import predict_finish_times

            assert predict_finish_times(q, c["t_now"], est) == c["finishes"]
    for c in P["estimate"]:
        est = S.PrefillThroughputEstimator(*c["est"])
        assert est.estimate_many(c["tokens"]).tolist() == c["out"]
    import warnings

    for c in P["synth"]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lut = S.synth_profile_from_anchors([tuple(a) for a in c["anchors"]], c["gamma"], bsz_buckets=c["bsz"],
                                               seq_buckets=c["seq"], prior_weight=c["weight"])
        assert lut._counts.tolist() == c["counts"]
        assert lut._sums.tolist() == [[float(x) for x in row] for row in c["sums"]]
        base = sorted((s2, float(u)) for b2, s2, u in c["anchors"] if b2 == 1)
        got = [S.decode_step_formula(base, c["gamma"], b2, s2) for b2, s2 in c["queries"]]
        assert got == c["formula"]


# ------------------------------------------------- known-answer behaviours --
def simple_profile(**kw):
    base = dict(decode_anchors=[(1, 8192, 10_000)], batch_growth=0.0, prefill_anchor=(10_000, 1_000_000))
    base.update(kw)
    return S.CostProfile(**base)


def test_single_request_timeline():
    w = [S.Request(id="a", arrival_time=0, input_len=100, output_len=2)]
    sim = S.Simulation(S.ClusterConfig(profile=simple_profile()), w, collect_events=True)
    rep = sim.run()
    r = sim.requests[0]
    assert r.t_prefill_finish == 10_000 and r.token_timestamps == [10_000, 20_000]
    assert rep.rows[0].ttft_us == 10_000 and rep.rows[0].mean_tpot_us == 10_000.0 and rep.rows[0].e2e_met


def test_empty_workload_and_validation():
    sim = S.Simulation(S.ClusterConfig(profile=simple_profile()), [], collect_events=True)
    rep = sim.run()
    assert rep.empty and rep.rows == [] and sim.events == []
    with pytest.raises(S.ConfigurationError):
        S.Simulation(S.ClusterConfig(kv_capacity_tokens=1100, profile=simple_profile()),
                     [S.Request(id="a", arrival_time=0, input_len=1000, output_len=200)])
    with pytest.raises(ValueError):
        S.Simulation(S.ClusterConfig(profile=simple_profile()),
                     [S.Request("a", 10, 5, 1), S.Request("b", 5, 5, 1)])
    with pytest.raises(S.ConfigurationError):
        S.ClusterConfig(prefill_policy="mystery")


def test_long_request_violates_ttft_alone():
    rep = S.run(S.ClusterConfig(profile=S.CostProfile()), [S.Request(id="L", arrival_time=0, input_len=131072, output_len=1)])
    assert rep.rows[0].ttft_us == 8_800_000 and not rep.rows[0].ttft_met


def test_kv_admission_blocks_then_drains():
    w = [S.Request(id="a", arrival_time=0, input_len=100, output_len=5),
         S.Request(id="b", arrival_time=1, input_len=100, output_len=5)]
    sim = S.Simulation(S.ClusterConfig(kv_capacity_tokens=105, profile=simple_profile()), w)
    sim.run()
    a, b = sim.requests
    assert a.t_first_token == 10_000 and b.t_first_token == 20_000
    assert b.token_timestamps[1] > a.token_timestamps[-1]


def test_transfer_delay_and_prefix_hits():
    sim = S.Simulation(S.ClusterConfig(transfer_base_us=500, transfer_per_token_us=1.0, profile=simple_profile()),
                       [S.Request(id="a", arrival_time=0, input_len=100, output_len=1)])
    sim.run()
    assert sim.requests[0].t_first_token == 10_000 + 500 + 100
    sim = S.Simulation(S.ClusterConfig(profile=simple_profile()),
                       [S.Request(id="a", arrival_time=0, input_len=100, output_len=1, prefix_hit_len=50)])
    sim.run()
    assert sim.requests[0].t_prefill_finish == 5_000


def test_worst_queue_wait():
    w = [S.Request(id="a", arrival_time=0, input_len=16_384, output_len=1),
         S.Request(id="b", arrival_time=1, input_len=100, output_len=1)]
    assert S.run(S.ClusterConfig(profile=simple_profile(), prefill_policy="fcfs"), w).worst_queue_wait_us == 1_638_399
    assert S.run(S.ClusterConfig(profile=simple_profile()), w[:1]).worst_queue_wait_us == 0


def test_noisy_decode_feeds_online_lut():
    sim = S.Simulation(S.ClusterConfig(profile=simple_profile(decode_noise_eps=0.3), seed=5),
                       [S.Request(id="a", arrival_time=0, input_len=100, output_len=30)])
    sim.run()
    assert sim.lut.observation_count(1, 8192) == 129
    assert sim.lut.lookup(1, 8192) != 10_000.0


def test_hol_blocking_acceptance():
    """Acceptance 1 (SPEC): FCFS meets 0/11 TTFTs, kairos-urgency 10/11 (all but L)."""
    prof = S.CostProfile(prefill_anchor=(139264, 9_200_400), prefill_gt_curve=[(8192, 400_400), (131072, 8_800_000)])
    w = [S.Request(id="L", arrival_time=0, input_len=131072, output_len=1)]
    w += [S.Request(id=f"S{k:02d}", arrival_time=100_000 * k, input_len=8192, output_len=1) for k in range(1, 11)]
    f = S.run(S.ClusterConfig(prefill_policy="fcfs", decode_policy="continuous", profile=prof), w)
    assert sum(r.ttft_met for r in f.rows) == 0
    k = S.run(S.ClusterConfig(prefill_policy="kairos-urgency", decode_policy="kairos-slack", profile=prof), w)
    met = {r.id for r in k.rows if r.ttft_met}
    assert len(met) == 10 and "L" not in met


def decode_loop(requests, lut, slo, policy):
    """Float-time decode-only loop with exact-LUT step costs (restated from SPEC acceptance 2/5)."""
    by_id = {r.id: r for r in requests}
    for r in requests:
        r.record_first_token(0.0)
    t = 0.0
    while True:
        active = [r for r in requests if r.n_gen < r.output_len - 1]
        if not active:
            return requests
        sel = S.DECODE_POLICIES[policy](active, t, slo, lut)
        batch = [by_id[i] for i in sel.batch]
        t += lut.lookup(len(batch), max(r.seq_len for r in batch))
        for r in batch:
            r.record_decode_token(t)


def test_decode_straggler_acceptance():
    slo = S.SLOConfig()
    pair = lambda: [S.Request(id="S", arrival_time=0, input_len=8192, output_len=200),
                    S.Request(id="L", arrival_time=0, input_len=131072, output_len=200)]
    anchors = [(1, 8192, 11_000), (1, 131072, 40_300)]
    cont = decode_loop(pair(), S.synth_profile_from_anchors(anchors, 0.03), slo, "continuous")
    cont_tps = S.decode_throughput(cont[0])
    assert cont_tps == pytest.approx(24.1, abs=0.1)
    adap = decode_loop(pair(), S.synth_profile_from_anchors(anchors, 0.03), slo, "kairos-slack")
    assert S.decode_throughput(adap[0]) >= 1.3 * cont_tps
    assert all(S.deadline_misses(r, slo) == 0 for r in adap)


def test_metric_known_answers():
    slo = S.SLOConfig()

    def finished(rid, times):
        r = S.Request(id=rid, arrival_time=0, input_len=100, output_len=len(times))
        r.record_first_token(times[0])
        for t in times[1:]:
            r.record_decode_token(t)
        return r

    assert S.ttft_metric(finished("a", [8_000_000]), slo) == (8_000_000, True)
    assert S.ttft_metric(finished("a", [8_800_000]), slo) == (8_800_000, False)
    assert S.tpot_metric(finished("a", [k * 50_000 for k in range(10)]), slo) == (50_000.0, True)
    assert S.deadline_misses(finished("a", [0, 60_000, 90_000]), slo) == 1
    assert S.decode_throughput(finished("a", [0, 40_300])) == pytest.approx(24.8, abs=0.05)
    assert S.decode_throughput(finished("a", [123])) is None


def test_policy_known_answers():
    lut = S.synth_profile_from_anchors([(1, 8192, 11_000), (1, 131072, 40_300)], 0.03)
    assert lut.lookup(1, 8192) == 11_000.0 and lut.lookup(2, 131072) == 41_509.0
    est = S.PrefillThroughputEstimator.seeded(3, 1_000)
    assert est.estimate_duration_us(1) == 334
    est = S.PrefillThroughputEstimator.seeded(10_000, 1_000_000)
    a, b = (S.Request(id=x, arrival_time=0, input_len=6000, output_len=1) for x in "ab")
    assert S.select_prefill_batch([b, a], 8192, 0, est, S.SLOConfig()).entries == [("a", 6000), ("b", 2192)]
    est = S.PrefillThroughputEstimator.seeded(131072, 8_800_000)
    A = S.Request(id="A", arrival_time=0, input_len=65536, output_len=1)
    B = S.Request(id="B", arrival_time=100_000, input_len=8192, output_len=1)
    assert S.select_prefill_batch([A, B], 8192, 100_000, est, S.SLOConfig()).entries == [("B", 8192)]
    from paper_2605_02329_b200.prefill_sched import predict_finish_times

    assert predict_finish_times([A, B], 100_000, est) == {"A": 4_500_000, "B": 5_050_000}

    def decoding(rid, inp, n_gen):
        r = S.Request(id=rid, arrival_time=0, input_len=inp, output_len=500)
        r.record_first_token(0)
        for k in range(n_gen):
            r.record_decode_token(k + 1)
        return r

    sel = S.select_decode_batch([decoding("L", 131072, 1), decoding("S", 8192, 1)], 28_491, S.SLOConfig(), lut)
    assert sel.batch == ["S"] and sel.delayed == ["L"] and not sel.fallback
    assert sel.s_min_us == pytest.approx(30_000.0)
    sel = S.select_decode_batch([decoding("r", 8192, 0)], 44_000, S.SLOConfig(), lut)
    assert sel.fallback and sel.batch == ["r"] and sel.s_min_us == pytest.approx(-5_000.0)
