"""Lowering of configs and traces to the packed C-ABI layout of include/slosim_b200.h.

Host marshalling only: traces become one concatenated SoA table, each distinct
CostProfile one ``slosim_profile_t`` (the synthesized LUT is computed on the
device by ``slosim_synth_profile``), each (trace, ClusterConfig, rate) point one
``slosim_instance_t``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from .config import DEFAULT_BSZ_BUCKETS, DEFAULT_SEQ_BUCKETS, ClusterConfig, CostProfile
from .domain import ConfigurationError
from .workload import TraceArrays

U64 = (1 << 64) - 1


def _check_buckets(buckets, name):
    if not buckets or any(b < 1 for b in buckets):
        raise ValueError(f"{name} buckets must be non-empty and >= 1")
    if any(a >= b for a, b in zip(buckets, buckets[1:])):
        raise ValueError(f"{name} buckets must be strictly increasing")


def _gpu_synth(P: _abi.Profile, anchors, gamma, weight):
    n = len(anchors)
    ab = np.array([int(a[0]) for a in anchors], np.int64)
    asq = np.array([int(a[1]) for a in anchors], np.int64)
    au = np.array([float(a[2]) for a in anchors], np.float64)
    rc = _abi.lib().slosim_synth_profile(
        ctypes.byref(P), n, ab.ctypes.data, asq.ctypes.data, au.ctypes.data, float(gamma), int(weight)
    )
    if rc != _abi.OK:
        raise ValueError(f"slosim_synth_profile failed ({rc})")


def fill_lut_fields(P: _abi.Profile, bsz_buckets, seq_buckets, sums, counts, prefix="lut"):
    """Write a [nb][ns] LUT into the 16x64 frame of the profile struct."""
    nb, ns = len(bsz_buckets), len(seq_buckets)
    fs = np.zeros((_abi.MAX_B, _abi.MAX_S), np.float64)
    fc = np.zeros((_abi.MAX_B, _abi.MAX_S), np.int32)
    fs[:nb, :ns] = np.asarray(sums, np.float64).reshape(nb, ns)
    fc[:nb, :ns] = np.asarray(counts, np.int64).reshape(nb, ns)
    ctypes.memmove(getattr(P, f"{prefix}_sums"), fs.ctypes.data, fs.nbytes)
    ctypes.memmove(getattr(P, f"{prefix}_counts"), fc.ctypes.data, fc.nbytes)


def profile_struct(cost: CostProfile, synth=None) -> _abi.Profile:
    """Resolve a CostProfile the way Simulation.__init__ / _GroundTruth do (engine.py:85-159)."""
    from .costmodel import load_profile

    P = _abi.Profile()
    if cost.profile_path is not None:
        lut, anchor = load_profile(cost.profile_path)
        bb, sb = list(lut.bsz_buckets), list(lut.seq_buckets)
        if len(bb) > _abi.MAX_B or len(sb) > _abi.MAX_S:
            raise ConfigurationError("LUT grid exceeds the device limits (16 x 64)")
        P.nb, P.ns = len(bb), len(sb)
        P.bsz_buckets[: len(bb)] = bb
        P.seq_buckets[: len(sb)] = sb
        fill_lut_fields(P, bb, sb, lut._sums, lut._counts, "lut")
        fill_lut_fields(P, bb, sb, lut._sums, lut._counts, "gt")
        P.gt_frozen = 1
        prefill_anchor = anchor
        est = anchor
        P.n_base = 0
    else:
        bb = list(DEFAULT_BSZ_BUCKETS) if cost.bsz_buckets is None else list(cost.bsz_buckets)
        sb = list(DEFAULT_SEQ_BUCKETS) if cost.seq_buckets is None else list(cost.seq_buckets)
        _check_buckets(bb, "bsz")
        _check_buckets(sb, "seq")
        if len(bb) > _abi.MAX_B or len(sb) > _abi.MAX_S:
            raise ConfigurationError("LUT grid exceeds the device limits (16 x 64)")
        if cost.batch_growth < 0:
            raise ValueError("batch_growth must be >= 0")
        if cost.prior_weight < 0:
            raise ValueError("prior_weight must be >= 0")
        base = sorted((int(s), float(us)) for b, s, us in cost.decode_anchors if b == 1)
        if not base:
            raise ValueError("need at least one anchor at bsz=1")
        if len(base) > _abi.MAX_BASE:
            raise ConfigurationError("too many decode anchors for the device (16)")
        P.nb, P.ns = len(bb), len(sb)
        P.bsz_buckets[: len(bb)] = bb
        P.seq_buckets[: len(sb)] = sb
        (synth or _gpu_synth)(P, list(cost.decode_anchors), cost.batch_growth, cost.prior_weight)
        P.n_base = len(base)
        for k, (s, us) in enumerate(base):
            P.base_x[k] = s
            P.base_y[k] = us
        P.gt_frozen = 0
        prefill_anchor = tuple(cost.prefill_anchor)
        est = prefill_anchor
    P.gamma = float(cost.batch_growth)
    P.noise_eps = float(cost.decode_noise_eps)
    P.est_tokens, P.est_busy_us = int(est[0]), int(est[1])
    if cost.prefill_gt_curve is not None:
        pts = sorted((int(t), int(d)) for t, d in cost.prefill_gt_curve)
        if not pts or any(t <= 0 or d <= 0 for t, d in pts):
            raise ConfigurationError("prefill_gt_curve points must be positive")
    else:
        pts = [(int(prefill_anchor[0]), int(prefill_anchor[1]))]
    curve = [(0, 0)] + pts
    if len(curve) > _abi.MAX_CURVE:
        raise ConfigurationError("prefill_gt_curve has too many points for the device (15)")
    P.n_curve = len(curve)
    for k, (x, y) in enumerate(curve):
        P.curve_x[k] = x
        P.curve_y[k] = y
    return P


def rng_state(seed: int):
    """numpy PCG64 state of default_rng(seed) (engine.py:225) as (hi, lo, inc_hi, inc_lo)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return (s >> 64) & U64, s & U64, (inc >> 64) & U64, inc & U64


class PackedBatch:
    """Host arrays of one batch, ready for slosim_run_batch_host or device upload."""

    def __init__(self, arrival, inp, out, hit, idr, profiles, instances, flags, n_rows, trace_words):
        self.arrival, self.inp, self.out, self.hit, self.idr = arrival, inp, out, hit, idr
        self.profiles = profiles  # ctypes array of Profile
        self.instances = instances  # structured numpy array (instance_dtype)
        self.flags = int(flags)
        self.n_rows = int(n_rows)
        self.trace_words = int(trace_words)
        self.summaries = np.zeros(len(instances), _abi.summary_dtype())
        self.rows = None
        if self.flags & _abi.F_ROWS:
            n = max(self.n_rows, 1)
            self.rows = {
                "ttft_us": np.zeros(n, np.int64), "mean_tpot_us": np.zeros(n, np.float64),
                "decode_tps": np.zeros(n, np.float64), "met_flags": np.zeros(n, np.uint8),
                "deadline_misses": np.zeros(n, np.int32), "t_prefill_finish": np.zeros(n, np.int64),
                "t_first_token": np.zeros(n, np.int64), "t_last_token": np.zeros(n, np.int64),
                "first_sched_us": np.zeros(n, np.int64),
            }
        self.trace_buf = np.zeros(max(self.trace_words, 1), np.int64) if self.trace_words else None
        self.lut_out_sums = self.lut_out_counts = None
        if self.flags & _abi.F_EXPORT_LUT:
            self.lut_out_sums = np.zeros((len(instances), _abi.CELLS), np.float64)
            self.lut_out_counts = np.zeros((len(instances), _abi.CELLS), np.int32)

    @property
    def n_instances(self) -> int:
        return int(len(self.instances))

    @property
    def n_requests(self) -> int:
        return int(self.instances["n_requests"].sum())

    def host_struct(self) -> _abi.Batch:
        b = _abi.Batch()
        b.traces = _abi.Traces(
            self.arrival.ctypes.data, self.inp.ctypes.data, self.out.ctypes.data, self.hit.ctypes.data,
            self.idr.ctypes.data, int(self.arrival.shape[0]),
        )
        b.profiles = ctypes.addressof(self.profiles)
        b.n_profiles = len(self.profiles)
        b.flags = self.flags
        b.instances = self.instances.ctypes.data
        b.n_instances = len(self.instances)
        b.summaries = self.summaries.ctypes.data
        if self.rows is not None:
            for k, v in self.rows.items():
                setattr(b.rows, k, v.ctypes.data)
            b.rows_capacity = len(self.rows["ttft_us"])
        b.trace_buf = self.trace_buf.ctypes.data if self.trace_buf is not None else None
        b.trace_buf_capacity = len(self.trace_buf) if self.trace_buf is not None else 0
        if self.lut_out_sums is not None:
            b.lut_out_sums = self.lut_out_sums.ctypes.data
            b.lut_out_counts = self.lut_out_counts.ctypes.data
        b.max_requests = int(self.instances["n_requests"].max()) if len(self.instances) else 0
        return b


class BatchBuilder:
    """Accumulates traces, profiles and instances into one PackedBatch."""

    def __init__(self, synth=None):
        self._synth = synth
        self._traces = []  # list of TraceArrays
        self._trace_off = []
        self._n_trace = 0
        self._profiles = []
        self._profile_ids = {}
        self._inst = []
        self._rows = 0
        self._words = 0

    def add_trace(self, tr: TraceArrays) -> int:
        self._traces.append(tr)
        self._trace_off.append(self._n_trace)
        self._n_trace += len(tr)
        return len(self._traces) - 1

    def add_profile(self, cost: CostProfile) -> int:
        # keyed by identity; the entry keeps `cost` alive so its id() cannot be recycled
        key = id(cost)
        if key not in self._profile_ids:
            self._profiles.append(profile_struct(cost, self._synth))
            self._profile_ids[key] = (cost, len(self._profiles) - 1)
        return self._profile_ids[key][1]

    def add_instance(self, trace_id: int, cluster: ClusterConfig, *, rescale: float | None = None,
                     trace_words: int = 0) -> int:
        pid = self.add_profile(cluster.profile)
        tr = self._traces[trace_id]
        n = len(tr)
        rec = np.zeros((), _abi.instance_dtype())
        rec["trace_offset"] = self._trace_off[trace_id]
        rec["n_requests"] = n
        rec["profile_id"] = pid
        rec["rescale_factor"] = float(rescale) if rescale is not None else 0.0
        rec["ttft_slo_us"] = int(cluster.slo.ttft_slo_us)
        rec["tpot_slo_us"] = int(cluster.slo.tpot_slo_us)
        rec["kv_capacity_tokens"] = int(cluster.kv_capacity_tokens)
        rec["transfer_base_us"] = int(cluster.transfer_base_us)
        rec["transfer_per_token_us"] = float(cluster.transfer_per_token_us)
        rec["chunk_budget"] = int(cluster.chunk_budget)
        rec["prefill_policy"] = _abi.PREFILL_IDS[cluster.prefill_policy]
        rec["decode_policy"] = _abi.DECODE_IDS[cluster.decode_policy]
        if cluster.profile.decode_noise_eps > 0:
            sh, sl, ih, il = rng_state(cluster.seed)
            rec["rng_state_hi"], rec["rng_state_lo"], rec["rng_inc_hi"], rec["rng_inc_lo"] = sh, sl, ih, il
        rec["row_offset"] = self._rows
        self._rows += n
        if trace_words:
            rec["trace_buf_offset"] = self._words
            rec["trace_buf_words"] = trace_words
            self._words += trace_words
        else:
            rec["trace_buf_offset"] = -1
            rec["trace_buf_words"] = 0
        self._inst.append(rec)
        return len(self._inst) - 1

    def build(self, flags: int = 0) -> PackedBatch:
        def cat(name, dt):
            if not self._traces:
                return np.zeros(1, dt)
            return np.ascontiguousarray(np.concatenate([getattr(t, name) for t in self._traces]).astype(dt))

        profiles = (_abi.Profile * max(len(self._profiles), 1))(*self._profiles)
        inst = np.array(self._inst, dtype=_abi.instance_dtype()) if self._inst else np.zeros(0, _abi.instance_dtype())
        return PackedBatch(
            cat("arrival_us", np.int64), cat("input_len", np.int32), cat("output_len", np.int32),
            cat("prefix_hit_len", np.int32), cat("id_rank", np.int32), profiles, inst, flags, self._rows,
            self._words,
        )


def trace_words_bound(tr: TraceArrays, chunk_budget: int) -> int:
    """Upper bound of event-trace words for one instance.

    Every prefill step but those ending in a partial chunk completes >= 1
    request, and a partial step consumes the whole budget, so prefill steps
    <= n + Σ(input - hit) / budget; decode steps <= Σ(output - 1).
    """
    n = len(tr)
    work = int(np.sum(tr.input_len.astype(np.int64) - tr.prefix_hit_len))
    psteps = n + -(-work // max(int(chunk_budget), 1))
    tokens = int(np.sum(tr.output_len.astype(np.int64) - 1))
    return 10 * n + 5 * psteps + (n + psteps) + 5 * tokens + tokens + 16
