"""Batched sweeps: the throughput path (``run_batch``) and the SURVEY Appendix B configs.

``run_batch`` is the call that replaces the reference's sequential
``for qps: for pair: Simulation(...).run()`` loop (cli.py:130-138): every
(trace, rate, SLO scale, policy pair) point becomes one instance of a single
device launch.  Instances are built vectorised (numpy structured arrays), so a
million-instance sweep packs in well under a second.

Device memory and streams come from PyTorch (plumbing only); the work is the
CUDA engine behind ``slosim_run_batch`` (include/slosim_b200.h).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi
from .config import ClusterConfig, CostProfile
from .pack import PackedBatch, profile_struct
from .workload import LongTailSpec, TraceArrays, longtail_arrays, longtail_arrays_device, rescale_factor

PAIRS_2 = [("fcfs", "continuous"), ("kairos-urgency", "kairos-slack")]
PAIRS_3 = [("fcfs", "continuous"), ("sjf", "continuous"), ("kairos-urgency", "kairos-slack")]
PAIRS_4 = [("fcfs", "continuous"), ("fcfs", "kairos-slack"), ("kairos-urgency", "continuous"),
           ("kairos-urgency", "kairos-slack")]
CONFIG1_RATES = [0.4, 0.7, 1.0, 1.3, 1.6, 1.9]
SWEEP_RATES = [round(0.10 + 0.05 * k, 10) for k in range(64)]
SWEEP_SLO_SCALES = [0.25 * j for j in range(1, 17)]


@dataclass
class Sweep:
    """A packed batch plus the coordinates of each instance."""

    packed: PackedBatch
    coords: np.ndarray  # structured: trace, rate, slo_scale, pair
    traces: list
    name: str


def _coords_dtype():
    return np.dtype([("trace", "<i4"), ("rate", "<f8"), ("slo_scale", "<f8"), ("pair", "<i4")])


def grid_batch(traces: list, rates, slo_scales, pairs, *, profile: CostProfile | None = None,
               cluster: ClusterConfig | None = None, flags: int = 0, synth=None, name: str = "grid",
               order: str = "pair-major", select=None) -> Sweep:
    """All (trace x rate x SLO scale x pair) instances in one batch.

    ``rates=None`` keeps the traces' own arrival times (no rescale).  ``select``
    optionally restricts to a slice/index array of the full grid (benchmark
    steps process a bounded slice of config 5).
    """
    cluster = cluster or ClusterConfig()
    profile = profile or cluster.profile
    P = profile_struct(profile, synth)
    profiles = (_abi.Profile * 1)(P)
    offs = np.zeros(len(traces), np.int64)
    n_tr = np.array([len(t) for t in traces], np.int64)
    offs[1:] = np.cumsum(n_tr)[:-1]
    rate_list = [None] if rates is None else list(rates)
    # rescale factors per (trace, rate): Python floats exactly as rescale_qps computes them
    fac = np.zeros((len(traces), len(rate_list)), np.float64)
    for ti, tr in enumerate(traces):
        for ri, q in enumerate(rate_list):
            fac[ti, ri] = 0.0 if q is None else rescale_factor(tr.arrival_us, q)
            if q is not None and not _rescale_order_ok(tr, fac[ti, ri]):
                raise ValueError("rescaled order differs from id order; rescale on the host instead")
    T, Rn, Sn, Pn = len(traces), len(rate_list), len(slo_scales), len(pairs)
    total = T * Rn * Sn * Pn
    idx = np.arange(total, dtype=np.int64) if select is None else np.asarray(select, np.int64)
    # decomposition: pair-major keeps same-policy instances adjacent (uniform warp work)
    p = idx % Pn
    s = (idx // Pn) % Sn
    r = (idx // (Pn * Sn)) % Rn
    t = idx // (Pn * Sn * Rn)
    inst = np.zeros(len(idx), _abi.instance_dtype())
    inst["trace_offset"] = offs[t]
    inst["n_requests"] = n_tr[t]
    inst["profile_id"] = 0
    inst["rescale_factor"] = fac[t, r]
    scales = np.asarray(slo_scales, np.float64)
    ttft = np.array([round(cluster.slo.ttft_slo_us * x) for x in scales], np.int64)
    tpot = np.array([round(cluster.slo.tpot_slo_us * x) for x in scales], np.int64)
    inst["ttft_slo_us"] = ttft[s]
    inst["tpot_slo_us"] = tpot[s]
    inst["kv_capacity_tokens"] = cluster.kv_capacity_tokens
    inst["transfer_base_us"] = cluster.transfer_base_us
    inst["transfer_per_token_us"] = cluster.transfer_per_token_us
    inst["chunk_budget"] = cluster.chunk_budget
    pp = np.array([_abi.PREFILL_IDS[a] for a, _ in pairs], np.int8)
    dp = np.array([_abi.DECODE_IDS[b] for _, b in pairs], np.int8)
    inst["prefill_policy"] = pp[p]
    inst["decode_policy"] = dp[p]
    rows = np.zeros(len(idx), np.int64)
    rows[1:] = np.cumsum(n_tr[t])[:-1]
    inst["row_offset"] = rows
    inst["trace_buf_offset"] = -1
    if profile.decode_noise_eps > 0:
        from .pack import rng_state

        sh, sl, ih, il = rng_state(cluster.seed)
        inst["rng_state_hi"], inst["rng_state_lo"], inst["rng_inc_hi"], inst["rng_inc_lo"] = sh, sl, ih, il
    cat = lambda name, dt: np.ascontiguousarray(np.concatenate([getattr(x, name) for x in traces]).astype(dt))
    packed = PackedBatch(cat("arrival_us", np.int64), cat("input_len", np.int32), cat("output_len", np.int32),
                         cat("prefix_hit_len", np.int32), cat("id_rank", np.int32), profiles, inst, flags,
                         int(n_tr[t].sum()), 0)
    coords = np.zeros(len(idx), _coords_dtype())
    coords["trace"] = t
    coords["rate"] = np.array([np.nan if q is None else q for q in rate_list], np.float64)[r]
    coords["slo_scale"] = scales[s]
    coords["pair"] = p
    return Sweep(packed, coords, traces, name)


def _rescale_order_ok(tr: TraceArrays, factor: float) -> bool:
    """Device rescale keeps position order iff ties of the rescaled arrivals are in id order."""
    idr = tr.id_rank
    if len(idr) < 2 or np.all(np.diff(idr) > 0):
        return True
    a = np.rint(tr.arrival_us.astype(np.float64) * factor).astype(np.int64)
    tie = a[1:] == a[:-1]
    return bool(np.all(idr[1:][tie] > idr[:-1][tie]))


# ----------------------------------------------------- SURVEY Appendix B ---
# gen="host": traces from numpy (the reference's own draws); gen="device": the same traces
# generated on the GPU by slosim_gen_longtail (bit-identical, tests/test_gpu_longtail.py).
def _traces(specs, gen: str) -> list:
    if gen == "device":
        return longtail_arrays_device(specs)
    if gen != "host":
        raise ValueError(f"gen must be 'host' or 'device', not {gen!r}")
    return [longtail_arrays(s) for s in specs]


def config1(gen: str = "host", **kw) -> Sweep:
    """gen_longtail(LongTailSpec()) x 6 CLI rates x 2 pairs (12 instances)."""
    base, = _traces([LongTailSpec()], gen)
    return grid_batch([base], CONFIG1_RATES, [1.0], PAIRS_2, name="config1", **kw)


def config2(gen: str = "host", **kw) -> Sweep:
    """One 100k-request trace at qps 1.0, kairos and fcfs pairs (2 instances)."""
    base, = _traces([LongTailSpec(n_requests=100_000, seed=2024, qps=1.0)], gen)
    return grid_batch([base], None, [1.0], PAIRS_2[::-1], name="config2", **kw)


def config3(gen: str = "host", **kw) -> Sweep:
    """Config-1 trace x 64 rates x 16 SLO scales x 3 pairs (3072 instances)."""
    base, = _traces([LongTailSpec()], gen)
    return grid_batch([base], SWEEP_RATES, SWEEP_SLO_SCALES, PAIRS_3, name="config3", **kw)


def split_round_robin(tr: TraceArrays, k: int) -> list:
    """Split a trace by position (i mod k) into k sub-traces, keeping ids and id ranks."""
    out = []
    for j in range(k):
        sel = np.arange(j, len(tr), k)
        ids = [tr.id_of(int(i)) for i in sel]
        rank = np.argsort(np.argsort(np.array(ids, dtype=object), kind="stable"), kind="stable").astype(np.int32)
        out.append(TraceArrays(tr.arrival_us[sel].copy(), tr.input_len[sel].copy(), tr.output_len[sel].copy(),
                               tr.prefix_hit_len[sel].copy(), rank, ids=ids))
    return out


def config4(seeds=range(256), n_requests=20_000, gen: str = "host", **kw) -> Sweep:
    """256 seeds x 20k requests at qps 4.0, split into 4 1P+1D pairs each, x 2 pairs (2048 instances)."""
    traces = []
    for tr in _traces([LongTailSpec(n_requests=n_requests, seed=int(s), qps=4.0) for s in seeds], gen):
        traces += split_round_robin(tr, 4)
    return grid_batch(traces, None, [1.0], PAIRS_2, name="config4", **kw)


def config5(seeds=range(256), select=None, gen: str = "host", **kw) -> Sweep:
    """256 seeds x 64 rates x 16 SLO scales x 4 pairs = 1,048,576 instances of 1k requests."""
    traces = _traces([LongTailSpec(seed=int(s)) for s in seeds], gen)
    return grid_batch(traces, SWEEP_RATES, SWEEP_SLO_SCALES, PAIRS_4, name="config5", select=select, **kw)


CONFIGS = {"config1": config1, "config2": config2, "config3": config3, "config4": config4, "config5": config5}


# ------------------------------------------------------------ device run ---
def schedule_order(instances: np.ndarray) -> np.ndarray:
    """Processing order for the persistent kernel's work queue.

    1. Group by decode policy (slack-guided first), then by prefill policy, so
       the warps resident on an SM at any moment run the same specialised
       engine loop and the same prefill handler, whose instruction working set
       then fits the SM's instruction cache (mixing policies on an SM costs up
       to 35%, tools/order_exp.py).
    2. Within a group, longest-first (LPT): the estimated cost is
       n_requests x arrival stretch (the rescale factor; a low target rate means
       many small decode steps), so the instances that finish last are short.
    """
    fac = instances["rescale_factor"].astype(np.float64)
    cost = instances["n_requests"].astype(np.float64) * np.where(fac > 0, fac, 1.0)
    dp = instances["decode_policy"].astype(np.int64)
    pp = instances["prefill_policy"].astype(np.int64)
    return np.lexsort((-cost, -pp, -dp)).astype(np.int64)


class DeviceBatch:
    """A packed batch resident in device memory (torch tensors as plumbing)."""

    def __init__(self, packed: PackedBatch, device="cuda", order: np.ndarray | None = None):
        import torch

        _abi.lib()
        self.packed = packed
        self.torch = torch
        t = lambda a: torch.from_numpy(np.array(a, copy=True)).to(device)
        self.arrival, self.inp, self.out = t(packed.arrival), t(packed.inp), t(packed.out)
        self.hit, self.idr = t(packed.hit), t(packed.idr)
        self.profiles = t(np.frombuffer(bytes(packed.profiles), np.uint8))
        self.instances = t(packed.instances.view(np.uint8))
        self.summaries = torch.zeros(packed.n_instances * ctypes.sizeof(_abi.Summary), dtype=torch.uint8,
                                     device=device)
        self.rows = None
        if packed.rows is not None:
            self.rows = {k: torch.zeros(v.shape, dtype=getattr(torch, str(v.dtype)), device=device)
                         for k, v in packed.rows.items()}
        self.struct = _abi.Batch()
        b = self.struct
        b.traces = _abi.Traces(self.arrival.data_ptr(), self.inp.data_ptr(), self.out.data_ptr(),
                               self.hit.data_ptr(), self.idr.data_ptr(), int(packed.arrival.shape[0]))
        b.profiles = self.profiles.data_ptr()
        b.n_profiles = len(packed.profiles)
        b.flags = packed.flags
        b.instances = self.instances.data_ptr()
        b.n_instances = packed.n_instances
        b.summaries = self.summaries.data_ptr()
        if self.rows is not None:
            for k, v in self.rows.items():
                setattr(b.rows, k, v.data_ptr())
            b.rows_capacity = int(self.rows["ttft_us"].numel())
        b.max_requests = int(packed.instances["n_requests"].max()) if packed.n_instances else 0
        self.order = t(schedule_order(packed.instances) if order is None else order)
        b.order = self.order.data_ptr()
        self._range_orders = {}

    def launch(self, stream=None) -> None:
        """Enqueue the engine on `stream` (default: torch's current stream)."""
        s = stream if stream is not None else self.torch.cuda.current_stream()
        rc = _abi.lib().slosim_run_batch(ctypes.byref(self.struct), ctypes.c_void_p(s.cuda_stream))
        if rc != _abi.OK:
            raise RuntimeError(f"slosim_run_batch failed ({rc}): {_abi.lib().slosim_last_error().decode()}")

    def launch_range(self, start: int, count: int, stream=None) -> None:
        """Enqueue the engine on instances [start, start+count) only (summaries land in place)."""
        s = stream if stream is not None else self.torch.cuda.current_stream()
        b = _abi.Batch.from_buffer_copy(self.struct)
        b.instances = self.instances.data_ptr() + start * ctypes.sizeof(_abi.Instance)
        b.summaries = self.summaries.data_ptr() + start * ctypes.sizeof(_abi.Summary)
        b.n_instances = count
        if start not in self._range_orders or self._range_orders[start][0] != count:
            o = schedule_order(self.packed.instances[start:start + count])
            self._range_orders[start] = (count, self.torch.from_numpy(o).to(self.order.device))
        b.order = self._range_orders[start][1].data_ptr()
        rc = _abi.lib().slosim_run_batch(ctypes.byref(b), ctypes.c_void_p(s.cuda_stream))
        if rc != _abi.OK:
            raise RuntimeError(f"slosim_run_batch failed ({rc}): {_abi.lib().slosim_last_error().decode()}")

    def fetch(self) -> np.ndarray:
        """Copy summaries (and rows) back into the packed batch; returns the summary array."""
        self.torch.cuda.synchronize()
        host = self.summaries.cpu().numpy().view(_abi.summary_dtype())
        self.packed.summaries[:] = host
        if self.rows is not None:
            for k, v in self.rows.items():
                self.packed.rows[k][:] = v.cpu().numpy()
        return self.packed.summaries


def run_batch(packed: PackedBatch, device="cuda") -> np.ndarray:
    """Run every instance on the GPU; returns the per-instance summary array."""
    db = DeviceBatch(packed, device)
    db.launch()
    return db.fetch()
