"""Decode-side policies (mirror of slosim/decode_sched.py), executed on the device.

``select_decode_batch`` runs ``slosim_select_decode``: the (seq_len, id)
ordering, full-batch fallback cost, min-slack reduction and the
ballot-driven speculative greedy scan of the batched engine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .costmodel import DecodeStepLUT, _check
from .domain import Request, SLOConfig, SimTime


@dataclass
class DecodeSelection:
    """Outcome of one decode scheduling decision (decode_sched.py:19-33)."""

    batch: list
    delayed: list
    predicted_step_time_us: float
    s_min_us: float
    fallback: bool = False
    admission_step_times_us: list = field(default_factory=list)


def compute_slack(r: Request, t_now: SimTime, slo: SLOConfig, lut: DecodeStepLUT, *,
                  step_cost_us: float | None = None) -> float:
    """Eq. 2 slack (decode_sched.py:36-57); the step cost comes from the device LUT."""
    if r.t_first_token is None:
        raise ValueError(f"{r.id}: slack undefined before the first token")
    if step_cost_us is None:
        step_cost_us = lut.lookup(1, r.seq_len)
    budget = slo.tpot_slo_us * (r.n_gen + 1)
    elapsed = t_now - r.t_first_token
    return budget - elapsed - step_cost_us


def _select(policy: str, active: list, t_now, slo: SLOConfig | None, lut: DecodeStepLUT) -> DecodeSelection:
    if not active:
        raise ValueError("active set must be non-empty")
    if policy == "kairos-slack":
        for r in active:
            if r.t_first_token is None:
                raise ValueError(f"{r.id}: slack undefined before the first token")
    n = len(active)
    seq = np.array([r.seq_len for r in active], np.int64)
    order = sorted(range(n), key=lambda k: active[k].id)
    idr = np.zeros(n, np.int32)
    idr[order] = np.arange(n, dtype=np.int32)
    ngen = np.array([r.n_gen for r in active], np.int64)
    tf = np.array([float(r.t_first_token) if r.t_first_token is not None else 0.0 for r in active], np.float64)
    bb, sb, sums, counts = lut._device_args()
    ob = np.zeros(n, np.int32)
    od = np.zeros(n, np.int32)
    ot = np.zeros(n, np.float64)
    nb_ = np.zeros(1, np.int32)
    nd_ = np.zeros(1, np.int32)
    fb = np.zeros(1, np.int32)
    pred = np.zeros(1, np.float64)
    smin = np.zeros(1, np.float64)
    tpot = int(slo.tpot_slo_us) if slo is not None else 1
    _check(_abi.lib().slosim_select_decode(
        _abi.DECODE_IDS[policy], n, seq.ctypes.data, idr.ctypes.data, ngen.ctypes.data, tf.ctypes.data, float(t_now),
        tpot, len(bb), bb.ctypes.data, len(sb), sb.ctypes.data, sums.ctypes.data, counts.ctypes.data,
        ob.ctypes.data, nb_.ctypes.data, od.ctypes.data, nd_.ctypes.data, ot.ctypes.data, pred.ctypes.data,
        smin.ctypes.data, fb.ctypes.data), "select_decode")
    k, d = int(nb_[0]), int(nd_[0])
    sel = DecodeSelection(
        batch=[active[int(i)].id for i in ob[:k]],
        delayed=[active[int(i)].id for i in od[:d]],
        predicted_step_time_us=float(pred[0]),
        s_min_us=float(smin[0]) if policy == "kairos-slack" else math.inf,
        fallback=bool(fb[0]),
        admission_step_times_us=[float(x) for x in ot[:k]] if (policy == "kairos-slack" and not fb[0]) else [],
    )
    return sel


def select_decode_batch(active: list, t_now: SimTime, slo: SLOConfig, lut: DecodeStepLUT) -> DecodeSelection:
    """Alg. 3 slack-guided greedy packing (decode_sched.py:60-111)."""
    return _select("kairos-slack", active, t_now, slo, lut)


def continuous_batching_select(active: list, lut: DecodeStepLUT) -> DecodeSelection:
    """Baseline: decode every active request (decode_sched.py:114-124)."""
    return _select("continuous", active, 0, None, lut)


DECODE_POLICIES = {
    "kairos-slack": select_decode_batch,
    "continuous": lambda active, t_now, slo, lut: continuous_batching_select(active, lut),
}
