"""Generate golden fixtures by running the REFERENCE slosim package (Python).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/slosim unmodified and records, for a set of
workloads x configs, the per-instance summary (met counts, p50/p90, worst wait,
step counts, byte-model counters), per-request rows, and the decision digest
computed from the reference's own event log with the digest definition shared
by the CUDA engine and the C oracle.  The
fixtures are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


def dstep(D, x):
    z = ((D ^ x) * 0x9E3779B97F4A7C15) & M64
    return z ^ (z >> 32)


def digest_from_events(events, pos_of):
    """Decision digest over the reference event log (PrefillStepDone/DecodeStepDone).

    Per prefill step: t, each (pos, take) in batch order, duration; per decode
    step: t, (sum of 32-bit member hashes << 32 | bsz), duration; each folded
    with dstep."""
    D = 0
    for ev in events:
        if ev["kind"] == "PrefillStepDone":
            D = dstep(D, ev["t_us"] ^ 0xA5A5A5A5A5A5A5A5)
            for rid, take in ev["detail"]["batch"]:
                D = dstep(D, (pos_of[rid] << 32) | take)
            D = dstep(D, ev["detail"]["duration_us"])
        elif ev["kind"] == "DecodeStepDone":
            s = 0
            for rid in ev["detail"]["batch"]:
                s = (s + (pos_of[rid] + 1) * 0x9E3779B1) & 0xFFFFFFFF
            D = dstep(D, ev["t_us"] ^ 0x5A5A5A5A5A5A5A5A)
            D = dstep(D, (s << 32) | ev["detail"]["bsz"])
            D = dstep(D, ev["detail"]["duration_us"])
    return D


def appendix_c_digest(events):
    """SURVEY Appendix C digest: SHA-256 over json.dumps of the step records."""
    h = hashlib.sha256()
    for ev in events:
        if ev["kind"] == "DecodeStepDone":
            h.update(json.dumps([ev["t_us"], sorted(ev["detail"]["batch"]), ev["detail"]["duration_us"]]).encode())
        elif ev["kind"] == "PrefillStepDone":
            h.update(json.dumps([ev["t_us"], ev["detail"]["batch"], ev["detail"]["duration_us"]]).encode())
    return h.hexdigest()[:16]


def byte_counters(slosim, sim_cls, cfg, workload):
    """V_dec, B_dec, V_pre by wrapping the reference registries."""
    from slosim import engine as E

    c = {"v_dec": 0, "b_dec": 0, "v_pre": 0, "max_queue": 0, "max_active": 0}
    pp = E.PREFILL_POLICIES[cfg.prefill_policy]
    dp = E.DECODE_POLICIES[cfg.decode_policy]

    def pw(queue, budget, t, est, slo):
        c["v_pre"] += len(queue)
        c["max_queue"] = max(c["max_queue"], len(queue))
        return pp(queue, budget, t, est, slo)

    def dw(active, t, slo, lut):
        c["v_dec"] += len(active)
        c["max_active"] = max(c["max_active"], len(active))
        sel = dp(active, t, slo, lut)
        c["b_dec"] += len(sel.batch)
        return sel

    sim = sim_cls(cfg, workload, collect_events=True)
    sim._prefill_policy = pw
    sim._decode_policy = dw
    return sim, c


def run_reference(slosim, cfg, workload):
    """Run one reference simulation; return a summary dict + per-request rows."""
    from slosim.engine import Simulation

    order = sorted(range(len(workload)), key=lambda k: (workload[k].arrival_time, workload[k].id))
    pos_of = {workload[k].id: p for p, k in enumerate(order)}
    try:
        sim, cnt = byte_counters(slosim, Simulation, cfg, workload)
    except slosim.ConfigurationError:
        return {"status": 3}
    try:
        rep = sim.run()
    except slosim.ConfigurationError:
        return {"status": 3}
    ev = sim.events
    tps = [r.decode_tps for r in rep.rows if r.decode_tps is not None]
    rows = {}
    for r in sim.requests:
        m = next(x for x in rep.rows if x.id == r.id)
        rows[pos_of[r.id]] = {
            "ttft_us": m.ttft_us, "mean_tpot_us": m.mean_tpot_us, "decode_tps": m.decode_tps,
            "flags": int(m.ttft_met) | (int(m.tpot_met) << 1) | (int(m.e2e_met) << 2),
            "deadline_misses": m.deadline_misses, "t_prefill_finish": r.t_prefill_finish,
            "t_first_token": r.t_first_token, "t_last_token": r.token_timestamps[-1] if r.token_timestamps else None,
            "first_sched_us": sim._first_sched.get(r.id),
        }
    return {
        "status": 0,
        "n": len(workload),
        "ttft_met": sum(x.ttft_met for x in rep.rows),
        "tpot_met": sum(x.tpot_met for x in rep.rows),
        "e2e_met": sum(x.e2e_met for x in rep.rows),
        "n_tps": len(tps),
        "tps_p50": rep.decode_tps_p50,
        "tps_p90": rep.decode_tps_p90,
        "worst_queue_wait_us": rep.worst_queue_wait_us,
        "prefill_steps": sum(1 for e in ev if e["kind"] == "PrefillStepDone"),
        "decode_steps": sum(1 for e in ev if e["kind"] == "DecodeStepDone"),
        "digest": str(digest_from_events(ev, pos_of)),
        "digest_c": appendix_c_digest(ev),
        "v_dec": cnt["v_dec"], "b_dec": cnt["b_dec"], "v_pre": cnt["v_pre"],
        "max_queue": cnt["max_queue"], "max_active": cnt["max_active"],
        "deadline_misses": sum(x.deadline_misses for x in rep.rows),
        "est_tokens": sim.estimator.total_tokens, "est_busy_us": sim.estimator.total_busy_us,
        "ttft_att": rep.ttft_attainment, "tpot_att": rep.tpot_attainment, "e2e_att": rep.e2e_attainment,
        "rows": rows,
    }


def wl_to_json(workload):
    return [[r.id, r.arrival_time, r.input_len, r.output_len, r.prefix_hit_len] for r in workload]


def cfg_to_json(cfg):
    p = cfg.profile
    return {
        "chunk_budget": cfg.chunk_budget, "kv_capacity_tokens": cfg.kv_capacity_tokens,
        "transfer_base_us": cfg.transfer_base_us, "transfer_per_token_us": cfg.transfer_per_token_us,
        "prefill_policy": cfg.prefill_policy, "decode_policy": cfg.decode_policy,
        "ttft_slo_us": cfg.slo.ttft_slo_us, "tpot_slo_us": cfg.slo.tpot_slo_us, "seed": cfg.seed,
        "profile": {
            "decode_anchors": [list(a) for a in p.decode_anchors], "batch_growth": p.batch_growth,
            "prior_weight": p.prior_weight, "bsz_buckets": p.bsz_buckets, "seq_buckets": p.seq_buckets,
            "prefill_anchor": list(p.prefill_anchor),
            "prefill_gt_curve": [list(x) for x in p.prefill_gt_curve] if p.prefill_gt_curve else None,
            "decode_noise_eps": p.decode_noise_eps,
        },
    }


def random_case(slosim, rng, k):
    """Random small workload + config covering every policy pair and knob."""
    n = rng.randrange(1, 41)
    wl = []
    for i in range(n):
        inp = rng.choice([rng.randrange(1, 3000), rng.randrange(1, 20000), rng.randrange(60000, 140000)])
        hit = rng.randrange(0, inp) if rng.random() < 0.2 else 0
        wl.append(slosim.Request(id=f"q{rng.randrange(10**6):06d}_{i}", arrival_time=rng.randrange(0, 4_000_000),
                                 input_len=inp, output_len=rng.choice([1, rng.randrange(1, 60), rng.randrange(1, 300)]),
                                 prefix_hit_len=hit))
    if rng.random() < 0.2:  # equal arrivals with ids out of position order
        for r in wl[: n // 2]:
            r.arrival_time = 1_000_000
    wl.sort(key=lambda r: r.arrival_time)  # engine only requires arrival order
    pp = ["fcfs", "sjf", "kairos-urgency"][k % 3]
    dp = ["continuous", "kairos-slack"][(k // 3) % 2]
    worst = max(r.input_len + r.output_len for r in wl)
    kv = worst + rng.choice([0, rng.randrange(0, 50_000), 2_000_000])
    anchors = rng.choice([
        [(1, 8192, 11_000), (1, 131072, 40_300)],
        [(1, 1024, 9_000), (1, 65536, 42_000)],
        [(1, 4096, 7_000), (1, 32768, 15_000), (1, 131072, 60_000), (4, 8192, 30_000)],
    ])
    bsz_b = rng.choice([None, None, [1, 3, 8, 20], [2, 4, 16, 64, 256]])
    seq_b = rng.choice([None, None, [1000, 10000, 100000, 200000], [8192 * k for k in range(1, 9)]])
    curve = rng.choice([None, None, [(8192, 400_400), (131072, 8_800_000)], [(5000, 300_000), (50000, 4_000_000)]])
    eps = rng.choice([0.0, 0.0, 0.0, 0.25])
    prof = slosim.CostProfile(decode_anchors=anchors, batch_growth=rng.choice([0.0, 0.03, 0.05]),
                              prior_weight=rng.choice([100, 100, 1, 7]), bsz_buckets=bsz_b, seq_buckets=seq_b,
                              prefill_anchor=rng.choice([(131072, 8_800_000), (10_000, 1_000_000), (139264, 9_200_400)]),
                              prefill_gt_curve=curve, decode_noise_eps=eps)
    cfg = slosim.ClusterConfig(
        chunk_budget=rng.choice([512, 2000, 4096, 8192, 8192]), kv_capacity_tokens=kv,
        transfer_base_us=rng.choice([0, 0, 150]), transfer_per_token_us=rng.choice([0.0, 0.0, 0.25, 1.0]),
        prefill_policy=pp, decode_policy=dp,
        slo=slosim.SLOConfig(ttft_slo_us=rng.choice([8_000_000, 2_000_000, 500_000]),
                             tpot_slo_us=rng.choice([50_000, 20_000, 100_000])),
        profile=prof, seed=rng.randrange(1000))
    return wl, cfg


def main():
    sys.path.insert(0, REF)
    import slosim

    if os.environ.get("GOLDEN_ONLY") == "policy":
        make_event_golden(slosim)
        make_policy_golden(slosim)
        return
    if os.environ.get("GOLDEN_ONLY") == "extra":
        make_extra_golden(slosim)
        return
    if os.environ.get("GOLDEN_ONLY") == "geo":
        make_geo_golden(slosim)
        return

    out = {"meta": {"reference": "slosim @ /root/reference/pkg/src", "numpy": __import__("numpy").__version__}}
    # --- config 1: 6 rates x 2 pairs on gen_longtail(LongTailSpec())
    base = slosim.gen_longtail(slosim.LongTailSpec())
    c1 = []
    for qps in [0.4, 0.7, 1.0, 1.3, 1.6, 1.9]:
        wl = slosim.rescale_qps(base, qps)
        for pp, dp in [("fcfs", "continuous"), ("kairos-urgency", "kairos-slack")]:
            cfg = slosim.ClusterConfig(prefill_policy=pp, decode_policy=dp)
            s = run_reference(slosim, cfg, wl)
            s.pop("rows")
            c1.append({"qps": qps, "pair": f"{pp}+{dp}", "summary": s})
            print("config1", qps, pp, s["e2e_met"], s["digest_c"], flush=True)
    out["config1"] = c1
    # --- random engine cases (all policy pairs, every knob)
    rng = random.Random(20260101)
    cases = []
    for k in range(int(os.environ.get("GOLDEN_CASES", "240"))):
        wl, cfg = random_case(slosim, rng, k)
        s = run_reference(slosim, cfg, wl)
        cases.append({"workload": wl_to_json(wl), "config": cfg_to_json(cfg), "summary": s})
    out["cases"] = cases
    print("cases", len(cases), sum(1 for c in cases if c["summary"]["status"] == 3), "config errors")
    path = os.path.join(HERE, "engine_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(out, f, sort_keys=True)
    print("wrote", path, os.path.getsize(path))
    make_event_golden(slosim)
    make_policy_golden(slosim)
    make_extra_golden(slosim)
    make_geo_golden(slosim)


def make_geo_golden(slosim):
    """Engine cases for the power-of-two LUT geometry path with arbitrary LUT values:
    fully populated file-backed profiles on bsz buckets 2^0..2^(nb-1) and seq buckets
    (j+1)*2^w (index arithmetic, exact power-of-two divisions) with fractional
    entries, frozen ground truth, noise, slack-guided and continuous decode, and
    synthesized profiles on reduced power-of-two grids (fast-forward paths)."""
    import tempfile

    rng = random.Random(4242)
    cases = []
    tmp = tempfile.mkdtemp()
    for k in range(40):
        burst = rng.random() < 0.5
        n = rng.randrange(40, 120) if burst else rng.randrange(20, 90)
        wl = []
        for i in range(n):
            inp = rng.choice([rng.randrange(1, 900), rng.randrange(1, 5000), rng.randrange(20000, 70000)])
            arr = rng.randrange(0, 60_000) if burst else rng.randrange(0, 4_000_000)
            wl.append(slosim.Request(id=f"g{i:03d}", arrival_time=arr, input_len=inp,
                                     output_len=rng.choice([1, rng.randrange(2, 80), rng.randrange(50, 300)]),
                                     prefix_hit_len=rng.randrange(0, inp) if rng.random() < 0.1 else 0))
        wl.sort(key=lambda r: r.arrival_time)
        nb = rng.randrange(2, 10)
        w = rng.choice([10, 12, 13, 14])
        ns = rng.randrange(2, min(64, (160_000 >> w) + 2))
        bszs = [1 << i for i in range(nb)]
        seqs = [(j + 1) << w for j in range(ns)]
        profile_json = None
        if k % 2 == 0:
            entries = [[float(rng.randrange(3_000, 60_000)) + rng.choice([0.0, 0.25, 0.5, 0.125]) for _ in seqs]
                       for _ in bszs]
            counts = [[rng.randrange(1, 50) for _ in seqs] for _ in bszs]
            profile_json = {"bsz_buckets": bszs, "seq_buckets": seqs, "entries_us": entries, "counts": counts,
                            "prefill_anchor": {"tokens": rng.choice([10_000, 131072]),
                                               "duration_us": rng.choice([1_000_000, 8_800_000])}}
            path = os.path.join(tmp, f"g{k}.json")
            with open(path, "w") as f:
                json.dump(profile_json, f)
            prof = slosim.CostProfile(profile_path=path, decode_noise_eps=rng.choice([0.0, 0.2]))
        else:
            prof = slosim.CostProfile(bsz_buckets=bszs, seq_buckets=seqs, decode_noise_eps=rng.choice([0.0, 0.0, 0.2]),
                                      prior_weight=rng.choice([1, 100]))
        pp = ["fcfs", "sjf", "kairos-urgency"][k % 3]
        dp = ["kairos-slack", "continuous", "kairos-slack"][(k // 3) % 3]
        cfg = slosim.ClusterConfig(prefill_policy=pp, decode_policy=dp, profile=prof, seed=rng.randrange(100),
                                   kv_capacity_tokens=rng.choice([2_000_000, 400_000]),
                                   chunk_budget=rng.choice([8192, 2048]),
                                   slo=slosim.SLOConfig(tpot_slo_us=rng.choice([50_000, 150_000, 400_000])))
        try:
            s = run_reference(slosim, cfg, wl)
        except slosim.ConfigurationError:
            continue
        cj = cfg_to_json(cfg)
        cj["profile"]["profile_json"] = profile_json
        cases.append({"workload": wl_to_json(wl), "config": cj, "summary": s})
    path = os.path.join(HERE, "geo_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(cases, f, sort_keys=True)
    print("wrote", path, len(cases), os.path.getsize(path))


def make_extra_golden(slosim):
    """Engine cases for the less common device paths: file-backed sparse LUTs
    (general lookup + frozen ground truth) and bursts with > 32 concurrently
    active decodes (memory-mode active set, register/memory switching)."""
    import tempfile

    rng = random.Random(99)
    cases = []
    tmp = tempfile.mkdtemp()
    for k in range(48):
        sparse = k % 2 == 0
        burst = rng.random() < 0.6
        n = rng.randrange(40, 130) if burst else rng.randrange(20, 90)
        wl = []
        for i in range(n):
            inp = rng.choice([rng.randrange(1, 900), rng.randrange(1, 5000), rng.randrange(20000, 70000)])
            if burst:
                inp = rng.randrange(1, 700)
            arr = rng.randrange(0, 50_000) if burst else rng.randrange(0, 3_000_000)
            wl.append(slosim.Request(id=f"x{i:03d}", arrival_time=arr, input_len=inp,
                                     output_len=rng.choice([1, rng.randrange(2, 80), rng.randrange(50, 400)])
                                     if not burst else rng.randrange(30, 300),
                                     prefix_hit_len=rng.randrange(0, inp) if rng.random() < 0.1 else 0))
        wl.sort(key=lambda r: r.arrival_time)
        profile_json = None
        if sparse:
            bszs = sorted(rng.sample(range(1, 80), rng.randrange(2, 7)))
            seqs = sorted(rng.sample(range(500, 150_000), rng.randrange(2, 9)))
            entries, counts = [], []
            for b in bszs:
                er, cr = [], []
                for sq in seqs:
                    if rng.random() < 0.6:
                        er.append(float(rng.randrange(3_000, 60_000)) + rng.choice([0.0, 0.25, 0.5]))
                        cr.append(rng.randrange(1, 50))
                    else:
                        er.append(0.0)
                        cr.append(0)
                entries.append(er)
                counts.append(cr)
            if not any(c for row in counts for c in row):
                counts[0][0] = 3
                entries[0][0] = 9_000.0
            profile_json = {"bsz_buckets": bszs, "seq_buckets": seqs, "entries_us": entries, "counts": counts,
                            "prefill_anchor": {"tokens": rng.choice([10_000, 131072]),
                                               "duration_us": rng.choice([1_000_000, 8_800_000])}}
            path = os.path.join(tmp, f"p{k}.json")
            with open(path, "w") as f:
                json.dump(profile_json, f)
            prof = slosim.CostProfile(profile_path=path, decode_noise_eps=rng.choice([0.0, 0.2]))
        else:
            prof = slosim.CostProfile(decode_noise_eps=rng.choice([0.0, 0.2]))
        pp = ["fcfs", "sjf", "kairos-urgency"][k % 3]
        dp = ["continuous", "kairos-slack"][(k // 3) % 2]
        cfg = slosim.ClusterConfig(prefill_policy=pp, decode_policy=dp, profile=prof, seed=rng.randrange(100),
                                   kv_capacity_tokens=rng.choice([2_000_000, 400_000, 150_000]),
                                   chunk_budget=rng.choice([8192, 2048]),
                                   slo=slosim.SLOConfig(tpot_slo_us=rng.choice([50_000, 150_000, 400_000])))
        try:
            s = run_reference(slosim, cfg, wl)
        except slosim.ConfigurationError:
            continue
        cj = cfg_to_json(cfg)
        cj["profile"]["profile_json"] = profile_json
        cases.append({"workload": wl_to_json(wl), "config": cj, "summary": s})
    path = os.path.join(HERE, "extra_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(cases, f, sort_keys=True)
    print("wrote", path, len(cases), "max_active", max(c["summary"].get("max_active", 0) for c in cases),
          os.path.getsize(path))


def make_event_golden(slosim):
    """Full reference event logs + token timestamps for the drop-in Simulation tests."""
    from slosim.engine import Simulation

    rng = random.Random(777)
    out = []
    for k in range(36):
        wl, cfg = random_case(slosim, rng, k)
        if rng.random() < 0.5:
            wl = wl[: rng.randrange(1, len(wl) + 1)]
        try:
            sim = Simulation(cfg, wl, collect_events=True)
            sim.run()
        except slosim.ConfigurationError:
            continue
        out.append({
            "workload": wl_to_json(wl), "config": cfg_to_json(cfg), "events": sim.events,
            "requests": {r.id: {"tokens": r.token_timestamps, "tpf": r.t_prefill_finish} for r in sim.requests},
            "lut_counts": sim.lut._counts, "lut_sums": sim.lut._sums,
            "estimator": [sim.estimator.total_tokens, sim.estimator.total_busy_us],
        })
    path = os.path.join(HERE, "events_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(out, f, sort_keys=True)
    print("wrote", path, len(out), os.path.getsize(path))


def _rand_lut(slosim, rng):
    bszs = sorted(rng.sample(range(1, 12), rng.randrange(1, 5)))
    seqs = sorted(rng.sample(range(100, 200_000), rng.randrange(1, 7)))
    lut = slosim.DecodeStepLUT(bsz_buckets=bszs, seq_buckets=seqs)
    for b in bszs:
        for sq in seqs:
            if rng.random() < 0.8:
                for _ in range(rng.randrange(1, 3)):
                    lut.update(b, sq, rng.randrange(1_000, 80_000))
    if lut.is_empty:
        lut.update(bszs[0], seqs[0], 5_000)
    return lut


def make_policy_golden(slosim):
    """Policy-level snapshot vectors: LUT lookups, decode/prefill selection, estimator, synth."""
    rng = random.Random(4711)
    lut_cases, dec_cases, pre_cases, synth_cases, est_cases = [], [], [], [], []
    for _ in range(150):
        lut = _rand_lut(slosim, rng)
        qs = [(rng.randrange(1, 14), rng.choice([rng.randrange(1, 260_000)] + lut.seq_buckets)) for _ in range(40)]
        lut_cases.append({"bsz": lut.bsz_buckets, "seq": lut.seq_buckets, "sums": lut._sums, "counts": lut._counts,
                          "queries": qs, "values": [lut.lookup(b, sq) for b, sq in qs]})
    slo = slosim.SLOConfig()
    for k in range(400):
        lut = _rand_lut(slosim, rng) if k % 2 else slosim.synth_profile_from_anchors(
            [(1, 8192, 11_000), (1, 131072, 40_300)], 0.03)
        active = []
        for i in range(rng.randrange(1, 12 if k % 3 else 45)):
            r = slosim.Request(id=f"d{rng.randrange(10**5)}_{i}", arrival_time=0,
                               input_len=rng.randrange(1, 150_000), output_len=200)
            r.record_first_token(0)
            for j in range(rng.randrange(0, 40)):
                r.record_decode_token(j + 1)
            active.append(r)
        t_now = rng.randrange(1, 2_000_000)
        for pol in ("kairos-slack", "continuous"):
            sel = slosim.DECODE_POLICIES[pol](active, t_now, slo, lut)
            dec_cases.append({
                "policy": pol, "bsz": lut.bsz_buckets, "seq": lut.seq_buckets, "sums": lut._sums,
                "counts": lut._counts, "t_now": t_now,
                "active": [[r.id, r.input_len, r.n_gen, r.t_first_token] for r in active],
                "batch": sel.batch, "delayed": sel.delayed, "pred": sel.predicted_step_time_us,
                "smin": None if math.isinf(sel.s_min_us) else sel.s_min_us, "fallback": sel.fallback,
                "times": sel.admission_step_times_us})
    for k in range(400):
        est = slosim.PrefillThroughputEstimator.seeded(rng.randrange(5_000, 200_000), rng.randrange(300_000, 9_000_000))
        q = []
        for i in range(rng.randrange(0, 50 if k % 4 else 300)):
            inp = rng.randrange(1, 60_000)
            hit = rng.randrange(0, inp) if rng.random() < 0.3 else 0
            done = rng.randrange(0, inp - hit + 1) if rng.random() < 0.3 else 0
            q.append(slosim.Request(id=f"p{rng.randrange(10**5)}_{i}", arrival_time=rng.randrange(0, 4_000_000),
                                    input_len=inp, output_len=1, prefix_hit_len=hit, prefill_done_tokens=done))
        budget = rng.choice([1, 100, 4096, 8192, 20000])
        t_now = rng.randrange(0, 3_000_000)
        for pol in ("kairos-urgency", "fcfs", "sjf"):
            b = slosim.PREFILL_POLICIES[pol](q, budget, t_now, est, slo)
            pre_cases.append({
                "policy": pol, "budget": budget, "t_now": t_now, "est": [est.total_tokens, est.total_busy_us],
                "queue": [[r.id, r.arrival_time, r.input_len, r.prefix_hit_len, r.prefill_done_tokens] for r in q],
                "entries": b.entries,
                "finishes": slosim.prefill_sched.predict_finish_times(q, t_now, est) if pol == "fcfs" else None})
    for _ in range(60):
        anchors = [(1, rng.randrange(500, 150_000), rng.randrange(1_000, 60_000)) for _ in range(rng.randrange(1, 5))]
        if rng.random() < 0.5:
            anchors.append((rng.randrange(2, 300), rng.randrange(500, 300_000), rng.randrange(1_000, 90_000)))
        gamma = rng.choice([0.0, 0.03, 0.05, 0.123])
        w = rng.choice([0, 1, 7, 100])
        bb = rng.choice([None, [1, 3, 8, 20]])
        sb = rng.choice([None, [1000, 10000, 100000, 200000]])
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lut = slosim.synth_profile_from_anchors(anchors, gamma, bsz_buckets=bb, seq_buckets=sb, prior_weight=w)
        qs = [(rng.randrange(1, 300), rng.randrange(1, 300_000)) for _ in range(20)]
        synth_cases.append({"anchors": anchors, "gamma": gamma, "weight": w, "bsz": bb, "seq": sb,
                            "sums": lut._sums, "counts": lut._counts,
                            "formula": [slosim.decode_step_formula(sorted((s2, float(u)) for b2, s2, u in anchors if b2 == 1),
                                                                   gamma, b2, s2) for b2, s2 in qs], "queries": qs})
    for _ in range(100):
        est = slosim.PrefillThroughputEstimator.seeded(rng.randrange(1, 10**9), rng.randrange(1, 10**11))
        toks = [rng.randrange(0, 10**6) for _ in range(30)]
        est_cases.append({"est": [est.total_tokens, est.total_busy_us], "tokens": toks,
                          "out": [est.estimate_duration_us(x) for x in toks]})
    path = os.path.join(HERE, "policy_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump({"lut": lut_cases, "decode": dec_cases, "prefill": pre_cases, "synth": synth_cases,
                   "estimate": est_cases}, f, sort_keys=True)
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
