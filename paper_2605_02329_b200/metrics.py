"""SLO-attainment metrics (mirror of slosim/metrics.py).

Per-request metrics and the aggregate are computed on the device: inside the
batched engine at each retirement, and for explicit token timestamps by the
``slosim_request_metrics`` kernel.  Serialisation helpers are host I/O.
"""

from __future__ import annotations

import csv
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .domain import Request, SLOConfig


@dataclass
class RequestMetrics:
    id: str
    ttft_us: int
    mean_tpot_us: float
    decode_tps: float | None
    ttft_met: bool
    tpot_met: bool
    e2e_met: bool
    deadline_misses: int


@dataclass
class MetricsReport:
    rows: list
    ttft_attainment: float
    tpot_attainment: float
    e2e_attainment: float
    decode_tps_p50: float | None
    decode_tps_p90: float | None
    worst_queue_wait_us: int
    empty: bool
    config: dict = field(default_factory=dict)
    seed: int = 0


def _device_metrics(reqs: list, slo: SLOConfig):
    """Run the device metrics kernels over finished requests (metrics.py:30-144)."""
    n = len(reqs)
    for r in reqs:
        if r.t_first_token is None:
            raise ValueError(f"{r.id}: no first token recorded")
    arr = np.array([r.arrival_time for r in reqs], np.float64)
    outl = np.array([r.output_len for r in reqs], np.int64)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r.token_timestamps) for r in reqs])
    ts = np.array([t for r in reqs for t in r.token_timestamps], np.float64) if n else np.zeros(1, np.float64)
    if ts.size == 0:
        ts = np.zeros(1, np.float64)
    ttft = np.zeros(max(n, 1), np.float64)
    tpot = np.zeros(max(n, 1), np.float64)
    tps = np.zeros(max(n, 1), np.float64)
    flags = np.zeros(max(n, 1), np.uint8)
    miss = np.zeros(max(n, 1), np.int32)
    agg = np.zeros(5, np.float64)
    rc = _abi.lib().slosim_request_metrics(n, arr.ctypes.data, outl.ctypes.data, off.ctypes.data, ts.ctypes.data,
                                           int(slo.ttft_slo_us), int(slo.tpot_slo_us), ttft.ctypes.data,
                                           tpot.ctypes.data, tps.ctypes.data, flags.ctypes.data, miss.ctypes.data,
                                           agg.ctypes.data)
    if rc != _abi.OK:
        raise ValueError("request metrics: invalid input")
    return ttft, tpot, tps, flags, miss, agg


def _row(rid, ttft, tpot, tps, flags, miss) -> RequestMetrics:
    ttft = float(ttft)
    return RequestMetrics(
        id=rid, ttft_us=int(ttft) if ttft.is_integer() else ttft, mean_tpot_us=float(tpot),
        decode_tps=None if math.isnan(tps) else float(tps),
        ttft_met=bool(flags & 1), tpot_met=bool(flags & 2), e2e_met=bool(flags & 4),
        deadline_misses=int(miss),
    )


def request_metrics(r: Request, slo: SLOConfig) -> RequestMetrics:
    ttft, tpot, tps, flags, miss, _ = _device_metrics([r], slo)
    return _row(r.id, ttft[0], tpot[0], tps[0], flags[0], miss[0])


def ttft_metric(r: Request, slo: SLOConfig):
    m = request_metrics(r, slo)
    return m.ttft_us, m.ttft_met


def tpot_metric(r: Request, slo: SLOConfig):
    if r.output_len == 1:
        return 0.0, True
    m = request_metrics(r, slo)
    return m.mean_tpot_us, m.tpot_met


def decode_throughput(r: Request):
    if r.output_len == 1:
        return None
    return request_metrics(r, SLOConfig()).decode_tps


def deadline_misses(r: Request, slo: SLOConfig) -> int:
    if r.t_first_token is None:
        raise ValueError(f"{r.id}: no first token recorded")
    return request_metrics(r, slo).deadline_misses


def nearest_rank(sorted_values: list, pct: float) -> float:
    """Nearest-rank percentile of an ascending list (metrics.py:87-92)."""
    if not sorted_values:
        raise ValueError("no values")
    rank = math.ceil(pct / 100.0 * len(sorted_values))
    return sorted_values[max(rank, 1) - 1]


def aggregate(rows: list, *, worst_queue_wait_us: int = 0, config: dict | None = None, seed: int = 0) -> MetricsReport:
    """Fold per-request rows into attainment fractions and percentiles (metrics.py:109-144)."""
    rows = sorted(rows, key=lambda row: row.id)
    if not rows:
        return MetricsReport(rows=[], ttft_attainment=1.0, tpot_attainment=1.0, e2e_attainment=1.0,
                             decode_tps_p50=None, decode_tps_p90=None, worst_queue_wait_us=worst_queue_wait_us,
                             empty=True, config=config or {}, seed=seed)
    n = len(rows)
    tps = sorted(row.decode_tps for row in rows if row.decode_tps is not None)
    return MetricsReport(
        rows=rows,
        ttft_attainment=sum(row.ttft_met for row in rows) / n,
        tpot_attainment=sum(row.tpot_met for row in rows) / n,
        e2e_attainment=sum(row.e2e_met for row in rows) / n,
        decode_tps_p50=nearest_rank(tps, 50) if tps else None,
        decode_tps_p90=nearest_rank(tps, 90) if tps else None,
        worst_queue_wait_us=worst_queue_wait_us, empty=False, config=config or {}, seed=seed,
    )


def report_to_dict(report: MetricsReport) -> dict:
    return {
        "rows": [
            {"id": row.id, "ttft_us": row.ttft_us, "mean_tpot_us": row.mean_tpot_us, "decode_tps": row.decode_tps,
             "ttft_met": row.ttft_met, "tpot_met": row.tpot_met, "e2e_met": row.e2e_met,
             "deadline_misses": row.deadline_misses}
            for row in report.rows
        ],
        "ttft_attainment": report.ttft_attainment,
        "tpot_attainment": report.tpot_attainment,
        "e2e_attainment": report.e2e_attainment,
        "decode_tps_p50": report.decode_tps_p50,
        "decode_tps_p90": report.decode_tps_p90,
        "worst_queue_wait_us": report.worst_queue_wait_us,
        "empty": report.empty,
        "config": report.config,
        "seed": report.seed,
    }


def report_from_dict(data: dict) -> MetricsReport:
    return MetricsReport(
        rows=[RequestMetrics(**row) for row in data["rows"]],
        ttft_attainment=data["ttft_attainment"], tpot_attainment=data["tpot_attainment"],
        e2e_attainment=data["e2e_attainment"], decode_tps_p50=data["decode_tps_p50"],
        decode_tps_p90=data["decode_tps_p90"], worst_queue_wait_us=data["worst_queue_wait_us"],
        empty=data["empty"], config=data["config"], seed=data["seed"],
    )


def report_to_json(report: MetricsReport) -> str:
    return json.dumps(report_to_dict(report), sort_keys=True, indent=2) + "\n"


def report_from_json(text: str) -> MetricsReport:
    return report_from_dict(json.loads(text))


PER_REQUEST_COLUMNS = ["id", "ttft_us", "mean_tpot_us", "decode_tps", "ttft_met", "tpot_met", "e2e_met",
                       "deadline_misses"]
SWEEP_COLUMNS = ["qps", "policy_pair", "ttft_att", "tpot_att", "e2e_att", "decode_tps_p50"]


def _fmt(value) -> str:
    if isinstance(value, bool):
        return "true" if value else "false"
    if value is None:
        return ""
    return repr(value) if isinstance(value, float) else str(value)


def write_csv_atomic(path: str, columns: list, rows: list) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w", newline="", encoding="utf-8") as f:
        writer = csv.writer(f)
        writer.writerow(columns)
        for row in rows:
            writer.writerow([_fmt(v) for v in row])
    os.replace(tmp, path)


def write_per_request_csv(path: str, report: MetricsReport) -> None:
    write_csv_atomic(path, PER_REQUEST_COLUMNS, [
        [row.id, row.ttft_us, row.mean_tpot_us, row.decode_tps, row.ttft_met, row.tpot_met, row.e2e_met,
         row.deadline_misses]
        for row in report.rows
    ])


def write_sweep_csv(path: str, rows: list) -> None:
    write_csv_atomic(path, SWEEP_COLUMNS, [[row[c] for c in SWEEP_COLUMNS] for row in rows])
