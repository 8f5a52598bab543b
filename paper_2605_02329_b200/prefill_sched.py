"""Prefill-side policies (mirror of slosim/prefill_sched.py), executed on the device.

Each policy call packs the queue snapshot and runs ``slosim_select_prefill``:
the warp-cooperative FCFS max-plus finish-time scan, urgency scoring and
ordered budget packing that the batched engine runs at every prefill step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from .costmodel import PrefillThroughputEstimator, _check
from .domain import ConfigurationError, Request, SLOConfig, SimTime


@dataclass
class PrefillBatch:
    """(request id, chunk tokens) pairs of one prefill step (prefill_sched.py:17-32)."""

    entries: list

    @property
    def total_tokens(self) -> int:
        return sum(tokens for _, tokens in self.entries)

    def __bool__(self) -> bool:
        return bool(self.entries)


def _id_ranks(queue):
    order = sorted(range(len(queue)), key=lambda k: queue[k].id)
    rank = np.zeros(len(queue), np.int32)
    rank[order] = np.arange(len(queue), dtype=np.int32)
    return rank


def _est_args(est):
    if not est.is_seeded or est.total_tokens == 0:
        raise ConfigurationError("prefill throughput estimator is unseeded")
    return int(est.total_tokens), int(est.total_busy_us)


def predict_finish_times(queue: list, t_now: SimTime, est: PrefillThroughputEstimator) -> dict:
    """Alg. 2 serial FCFS walk (prefill_sched.py:39-56) as a device max-plus scan."""
    if not queue:
        return {}
    tok, busy = _est_args(est)
    order = sorted(queue, key=lambda r: (r.arrival_time, r.id))
    arr = np.array([r.arrival_time for r in order], np.int64)
    rem = np.array([r.remaining_prefill_tokens for r in order], np.int64)
    out = np.zeros(len(order), np.int64)
    _check(_abi.lib().slosim_predict_finish(len(order), arr.ctypes.data, rem.ctypes.data, int(t_now), tok, busy,
                                            out.ctypes.data), "predict_finish_times")
    return {r.id: int(f) for r, f in zip(order, out)}


def predict_prefill_finish_time(queue: list, r: Request, t_now: SimTime, est: PrefillThroughputEstimator) -> SimTime:
    finishes = predict_finish_times(queue, t_now, est)
    if r.id not in finishes:
        raise ValueError(f"request {r.id!r} is not in the queue")
    return finishes[r.id]


def urgency(r: Request, predicted_finish: SimTime, slo: SLOConfig) -> float:
    """Fraction of the TTFT budget left (prefill_sched.py:68-74); scalar API helper."""
    slack = slo.ttft_slo_us - (predicted_finish - r.arrival_time)
    return slack / slo.ttft_slo_us


def normalized_urgency(r: Request, predicted_finish: SimTime, slo: SLOConfig) -> float:
    """Urgency per prompt token (prefill_sched.py:77-79, Eq. 1); scalar API helper."""
    return urgency(r, predicted_finish, slo) / r.input_len


def _select(policy: str, queue: list, budget: int, t_now: SimTime = 0, est=None, slo=None) -> PrefillBatch:
    if budget < 1:
        raise ValueError("chunk budget must be >= 1")
    if not queue:
        return PrefillBatch([])
    pid = _abi.PREFILL_IDS[policy]
    tok, busy = _est_args(est) if pid == _abi.PREFILL_IDS["kairos-urgency"] else (1, 1)
    ttft = int(slo.ttft_slo_us) if slo is not None else 1
    n = len(queue)
    arr = np.array([r.arrival_time for r in queue], np.int64)
    inp = np.array([r.input_len for r in queue], np.int32)
    rem = np.array([r.remaining_prefill_tokens for r in queue], np.int64)
    idr = _id_ranks(queue)
    oi = np.zeros(n, np.int32)
    ot = np.zeros(n, np.int64)
    no = np.zeros(1, np.int32)
    _check(_abi.lib().slosim_select_prefill(pid, n, arr.ctypes.data, inp.ctypes.data, rem.ctypes.data,
                                            idr.ctypes.data, int(budget), int(t_now), tok, busy, ttft,
                                            oi.ctypes.data, ot.ctypes.data, no.ctypes.data, None), "select_prefill")
    k = int(no[0])
    return PrefillBatch([(queue[int(oi[e])].id, int(ot[e])) for e in range(k)])


def select_prefill_batch(queue: list, budget: int, t_now: SimTime, est: PrefillThroughputEstimator,
                         slo: SLOConfig) -> PrefillBatch:
    """Urgency-ordered budget packing (prefill_sched.py:109-127)."""
    return _select("kairos-urgency", queue, budget, t_now, est, slo)


def fcfs_select_prefill(queue: list, budget: int) -> PrefillBatch:
    return _select("fcfs", queue, budget)


def sjf_select_prefill(queue: list, budget: int) -> PrefillBatch:
    return _select("sjf", queue, budget)


PREFILL_POLICIES = {
    "kairos-urgency": select_prefill_batch,
    "fcfs": lambda queue, budget, t_now, est, slo: fcfs_select_prefill(queue, budget),
    "sjf": lambda queue, budget, t_now, est, slo: sjf_select_prefill(queue, budget),
}
