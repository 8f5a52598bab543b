"""Simulation / run — drop-in for slosim/engine.py, executed by the CUDA engine.

``Simulation(config, workload).run()`` validates exactly as the reference
(engine.py:198-246), packs the workload as a one-instance batch and runs it on
the device through ``slosim_run_batch_host`` (include/slosim_b200.h).  The
device writes per-request rows, an event trace, the final LUT and estimator;
this module turns them back into the reference's Python-side state:
``sim.requests`` (token timestamps, phases), ``sim.events``, ``sim.lut``,
``sim.estimator`` and the ``MetricsReport``.
"""

from __future__ import annotations

import copy
import ctypes
import math

import numpy as np

from . import _abi
from .config import ClusterConfig, CostProfile  # noqa: F401  (re-export, engine.py API)
from .costmodel import DecodeStepLUT, PrefillThroughputEstimator
from .domain import ConfigurationError, Phase, Request
from .metrics import MetricsReport, RequestMetrics, aggregate
from .pack import BatchBuilder, trace_words_bound
from .workload import trace_arrays_from_requests


class EngineError(RuntimeError):
    """The device engine reported an internal failure."""


def _validate(workload: list) -> None:
    for a, b in zip(workload, workload[1:]):
        if b.arrival_time < a.arrival_time:
            raise ValueError("workload must be sorted by arrival_time")
    ids = [r.id for r in workload]
    if len(set(ids)) != len(ids):
        raise ValueError("workload ids must be unique")
    for r in workload:
        if r.phase != Phase.QUEUED or r.prefill_done_tokens or r.n_gen or r.token_timestamps:
            raise ValueError(f"workload request {r.id!r} is not pristine")


def run_packed(packed) -> None:
    """Run a PackedBatch on the device with host buffers (copies in and out)."""
    b = packed.host_struct()
    ms = ctypes.c_float(0.0)
    rc = _abi.lib().slosim_run_batch_host(ctypes.byref(b), ctypes.byref(ms))
    if rc != _abi.OK:
        raise EngineError(f"slosim_run_batch_host failed ({rc}): {_abi.lib().slosim_last_error().decode()}")
    packed.device_ms = float(ms.value)


def decode_trace(words: np.ndarray):
    """Split an event-trace buffer into records (see include/slosim_b200.h)."""
    recs = []
    k = 0
    n = len(words)
    while k < n:
        kind = int(words[k])
        if kind == _abi.EV_END:
            break
        if kind in (_abi.EV_ARRIVAL, _abi.EV_TRANSFER_DONE):
            recs.append((kind, int(words[k + 1]), int(words[k + 2])))
            k += 3
        elif kind == _abi.EV_ADMIT:
            recs.append((kind, int(words[k + 1]), int(words[k + 2]), int(words[k + 3])))
            k += 4
        elif kind == _abi.EV_PREFILL_DONE:
            m = int(words[k + 3])
            ent = [(int(w) >> 32, int(w) & 0xFFFFFFFF) for w in words[k + 4:k + 4 + m]]
            recs.append((kind, int(words[k + 1]), int(words[k + 2]), ent))
            k += 4 + m
        elif kind == _abi.EV_DECODE_DONE:
            bsz = int(words[k + 3])
            mem = [int(w) for w in words[k + 5:k + 5 + bsz]]
            recs.append((kind, int(words[k + 1]), int(words[k + 2]), bsz, int(words[k + 4]), mem))
            k += 5 + bsz
        else:
            raise EngineError(f"corrupt event trace (kind {kind} at word {k})")
    return recs


def check_config(config: ClusterConfig, workload: list):
    """The refusals of Simulation.__init__ (engine.py:218-232), in the same order.

    Returns the initial (DecodeStepLUT, PrefillThroughputEstimator); raises ConfigurationError.
    """
    lut = config.profile.build_lut()
    if lut.is_empty:
        raise ConfigurationError("decode LUT has no populated entries")
    est = config.profile.build_estimator()
    if config.profile.profile_path is None and not any(a[0] == 1 for a in config.profile.decode_anchors):
        raise ConfigurationError("decode anchors need at least one bsz=1 entry")
    worst = max((r.input_len + r.output_len for r in workload), default=0)
    if worst > config.kv_capacity_tokens:
        raise ConfigurationError(
            f"kv_capacity_tokens={config.kv_capacity_tokens} cannot hold the "
            f"largest request reservation ({worst} tokens)"
        )
    return lut, est


class Simulation:
    """One deterministic run of a workload against a cluster configuration (engine.py:195-413)."""

    def __init__(self, config: ClusterConfig, workload: list, *, collect_events: bool = False) -> None:
        self.config = config
        _validate(workload)
        self.requests = copy.deepcopy(workload)
        self.lut, self.estimator = check_config(config, self.requests)
        self.events = [] if collect_events else None
        self._ran = False

    def run(self) -> MetricsReport:
        cfg = self.config
        n = len(self.requests)
        if n == 0:
            return aggregate([], worst_queue_wait_us=0, config=cfg.to_echo_dict(), seed=cfg.seed)
        tr = trace_arrays_from_requests(self.requests)
        bb = BatchBuilder()
        tid = bb.add_trace(tr)
        words = trace_words_bound(tr, cfg.chunk_budget)
        bb.add_instance(tid, cfg, trace_words=words)
        packed = bb.build(_abi.F_ROWS | _abi.F_EXPORT_LUT)
        run_packed(packed)
        s = packed.summaries[0]
        if s["status"] == _abi.ECONFIG:
            raise ConfigurationError("device engine refused the configuration")
        if s["status"] != _abi.OK:
            raise EngineError(f"device engine status {int(s['status'])}")
        by_pos = {tr.id_of(p): p for p in range(n)}
        self._restore(tr, packed, by_pos)
        R = packed.rows
        rows = []
        for r in self.requests:
            p = by_pos[r.id]
            tps = float(R["decode_tps"][p])
            f = int(R["met_flags"][p])
            rows.append(RequestMetrics(
                id=r.id, ttft_us=int(R["ttft_us"][p]), mean_tpot_us=float(R["mean_tpot_us"][p]),
                decode_tps=None if math.isnan(tps) else tps, ttft_met=bool(f & 1), tpot_met=bool(f & 2),
                e2e_met=bool(f & 4), deadline_misses=int(R["deadline_misses"][p]),
            ))
        rows.sort(key=lambda row: row.id)
        self._first_sched = {r.id: int(R["first_sched_us"][by_pos[r.id]]) for r in self.requests}
        return MetricsReport(
            rows=rows,
            ttft_attainment=int(s["ttft_met"]) / n,
            tpot_attainment=int(s["tpot_met"]) / n,
            e2e_attainment=int(s["e2e_met"]) / n,
            decode_tps_p50=None if int(s["n_tps"]) == 0 else float(s["tps_p50"]),
            decode_tps_p90=None if int(s["n_tps"]) == 0 else float(s["tps_p90"]),
            worst_queue_wait_us=int(s["worst_queue_wait_us"]),
            empty=False,
            config=cfg.to_echo_dict(),
            seed=cfg.seed,
        )

    def _restore(self, tr, packed, by_pos) -> None:
        events, lut, est = restore_state(self.requests, tr, packed, 0, self.lut.bsz_buckets, self.lut.seq_buckets)
        if self.events is not None:
            self.events = events
        self.lut = lut
        self.estimator = est


def restore_state(requests: list, tr, packed, inst: int, bsz_buckets, seq_buckets):
    """Rebuild reference-side state of instance `inst` from device outputs.

    Mutates `requests` (token timestamps, prefill progress, phase) and returns
    (events, final DecodeStepLUT, final PrefillThroughputEstimator), the
    reference's Simulation.events / .lut / .estimator (engine.py:234-257).
    """
    n = len(tr)
    by_pos = {tr.id_of(p): p for p in range(n)}
    reqs_by_pos = [None] * n
    orig_index = {}
    for k, r in enumerate(requests):
        reqs_by_pos[by_pos[r.id]] = r
        orig_index[r.id] = k
    R = packed.rows
    off = int(packed.instances[inst]["trace_buf_offset"])
    words = int(packed.instances[inst]["trace_buf_words"])
    if int(packed.summaries[inst]["status"]) & 0x100:
        raise EngineError("event trace buffer overflow")
    recs = decode_trace(packed.trace_buf[off:off + words])
    row0 = int(packed.instances[inst]["row_offset"])
    ngen = [0] * n
    events = []
    for rec in recs:
        kind, t = rec[0], rec[1]
        if kind == _abi.EV_ARRIVAL:
            events.append({"t_us": t, "kind": "Arrival", "req": tr.id_of(rec[2]), "detail": {}})
        elif kind == _abi.EV_TRANSFER_DONE:
            events.append({"t_us": t, "kind": "TransferDone", "req": tr.id_of(rec[2]), "detail": {}})
        elif kind == _abi.EV_ADMIT:
            r = reqs_by_pos[rec[2]]
            r.record_first_token(rec[3])
            events.append({"t_us": t, "kind": "Admit", "req": r.id, "detail": {"first_token_us": rec[3]}})
        elif kind == _abi.EV_PREFILL_DONE:
            events.append({"t_us": t, "kind": "PrefillStepDone", "req": None,
                           "detail": {"batch": [[tr.id_of(p), take] for p, take in rec[3]], "duration_us": rec[2]}})
        elif kind == _abi.EV_DECODE_DONE:
            # selection.batch order: ascending (seq_len, id) at step start (decode_sched.py:74)
            mem = sorted(rec[5], key=lambda p: (int(tr.input_len[p]) + ngen[p], tr.id_of(p)))
            for p in mem:
                reqs_by_pos[p].record_decode_token(t)
                ngen[p] += 1
            events.append({"t_us": t, "kind": "DecodeStepDone", "req": None,
                           "detail": {"batch": [tr.id_of(p) for p in mem], "bsz": rec[3], "max_seq": rec[4],
                                      "duration_us": rec[2]}})
    # arrivals at one instant are logged in workload order (engine.py:262-263)
    i = 0
    while i < len(events):
        j = i
        while j < len(events) and events[j]["kind"] == "Arrival" and events[j]["t_us"] == events[i]["t_us"]:
            j += 1
        if j - i > 1:
            events[i:j] = sorted(events[i:j], key=lambda e: orig_index[e["req"]])
        i = max(j, i + 1)
    for p in range(n):
        r = reqs_by_pos[p]
        r.prefill_done_tokens = r.input_len - r.prefix_hit_len
        if R is not None:
            r.t_prefill_finish = int(R["t_prefill_finish"][row0 + p])
        r.phase = Phase.FINISHED
    lut = DecodeStepLUT(bsz_buckets, seq_buckets)
    if packed.lut_out_sums is not None:
        nb, ns = len(lut.bsz_buckets), len(lut.seq_buckets)
        fs = packed.lut_out_sums[inst].reshape(_abi.MAX_B, _abi.MAX_S)
        fc = packed.lut_out_counts[inst].reshape(_abi.MAX_B, _abi.MAX_S)
        lut._sums[:, :] = fs[:nb, :ns]
        lut._counts[:, :] = fc[:nb, :ns]
    s = packed.summaries[inst]
    est = PrefillThroughputEstimator(int(s["est_tokens"]), int(s["est_busy_us"]))
    return events, lut, est


def run(config: ClusterConfig, workload: list, *, collect_events: bool = False) -> MetricsReport:
    """Run one simulation to quiescence and return its metrics report (engine.py:416-420)."""
    return Simulation(config, workload, collect_events=collect_events).run()
