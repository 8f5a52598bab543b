"""ctypes mirror of include/slosim_b200.h and the loader of the CUDA library.

The library is built in-tree (``paper_2605_02329_b200/libslosim_b200.so``) by
``__graft_entry__.build()``.  There is no CPU fallback: if the library or a
CUDA device is missing, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int8, c_int32, c_int64, c_uint64, c_void_p

MAX_B = 16
MAX_S = 64
MAX_CURVE = 16
MAX_BASE = 16
CELLS = MAX_B * MAX_S

OK = 0
EINVAL = 2
ECONFIG = 3
ECUDA = 4
ENOMEM = 5
ERANGE = 6

DRAW_RAW, DRAW_RANDOM, DRAW_STD_EXPONENTIAL, DRAW_EXPONENTIAL, DRAW_STD_NORMAL, DRAW_LOGNORMAL, DRAW_INTEGERS = range(7)

PREFILL_IDS = {"fcfs": 0, "sjf": 1, "kairos-urgency": 2}
DECODE_IDS = {"continuous": 0, "kairos-slack": 1}

EV_ARRIVAL, EV_TRANSFER_DONE, EV_PREFILL_DONE, EV_DECODE_DONE, EV_ADMIT, EV_END = range(6)

F_ROWS = 1
F_EXPORT_LUT = 2
F_ALWAYS_LUT = 4


class Profile(ctypes.Structure):
    _fields_ = [
        ("nb", c_int32),
        ("ns", c_int32),
        ("bsz_buckets", c_int32 * MAX_B),
        ("seq_buckets", c_int32 * MAX_S),
        ("lut_sums", c_double * CELLS),
        ("lut_counts", c_int32 * CELLS),
        ("est_tokens", c_int64),
        ("est_busy_us", c_int64),
        ("n_curve", c_int32),
        ("_pad0", c_int32),
        ("curve_x", c_int64 * MAX_CURVE),
        ("curve_y", c_int64 * MAX_CURVE),
        ("n_base", c_int32),
        ("gt_frozen", c_int32),
        ("base_x", c_int64 * MAX_BASE),
        ("base_y", c_double * MAX_BASE),
        ("gamma", c_double),
        ("noise_eps", c_double),
        ("gt_sums", c_double * CELLS),
        ("gt_counts", c_int32 * CELLS),
    ]


class Instance(ctypes.Structure):
    _fields_ = [
        ("trace_offset", c_int64),
        ("n_requests", c_int32),
        ("profile_id", c_int32),
        ("rescale_factor", c_double),
        ("ttft_slo_us", c_int64),
        ("tpot_slo_us", c_int64),
        ("kv_capacity_tokens", c_int64),
        ("transfer_base_us", c_int64),
        ("transfer_per_token_us", c_double),
        ("chunk_budget", c_int32),
        ("prefill_policy", c_int8),
        ("decode_policy", c_int8),
        ("_pad1", c_int8 * 2),
        ("rng_state_hi", c_uint64),
        ("rng_state_lo", c_uint64),
        ("rng_inc_hi", c_uint64),
        ("rng_inc_lo", c_uint64),
        ("row_offset", c_int64),
        ("trace_buf_offset", c_int64),
        ("trace_buf_words", c_int64),
    ]


class Traces(ctypes.Structure):
    _fields_ = [
        ("arrival_us", c_void_p),
        ("input_len", c_void_p),
        ("output_len", c_void_p),
        ("prefix_hit_len", c_void_p),
        ("id_rank", c_void_p),
        ("n_total", c_int64),
    ]


class LongTailSpec(ctypes.Structure):
    """slosim_longtail_spec_t: LongTailSpec (workload.py:52-85) + output offset."""

    _fields_ = [
        ("qps", c_double),
        ("n_requests", c_int64),
        ("short_len_log_mean", c_double),
        ("short_len_log_sigma", c_double),
        ("p_long", c_double),
        ("long_len_min", c_int64),
        ("long_len_max", c_int64),
        ("out_len_log_mean", c_double),
        ("out_len_log_sigma", c_double),
        ("seed", c_uint64),
        ("offset", c_int64),
    ]


class Summary(ctypes.Structure):
    _fields_ = [
        ("status", c_int32),
        ("n", c_int32),
        ("ttft_met", c_int32),
        ("tpot_met", c_int32),
        ("e2e_met", c_int32),
        ("n_tps", c_int32),
        ("tps_p50", c_double),
        ("tps_p90", c_double),
        ("worst_queue_wait_us", c_int64),
        ("prefill_steps", c_int64),
        ("decode_steps", c_int64),
        ("digest", c_uint64),
        ("v_dec", c_int64),
        ("b_dec", c_int64),
        ("v_pre", c_int64),
        ("deadline_misses", c_int64),
        ("t_end_us", c_int64),
        ("est_tokens", c_int64),
        ("est_busy_us", c_int64),
        ("max_queue", c_int32),
        ("max_active", c_int32),
        ("sim_cycles", c_int64),
    ]


class Rows(ctypes.Structure):
    _fields_ = [
        ("ttft_us", c_void_p),
        ("mean_tpot_us", c_void_p),
        ("decode_tps", c_void_p),
        ("met_flags", c_void_p),
        ("deadline_misses", c_void_p),
        ("t_prefill_finish", c_void_p),
        ("t_first_token", c_void_p),
        ("t_last_token", c_void_p),
        ("first_sched_us", c_void_p),
    ]


class Batch(ctypes.Structure):
    _fields_ = [
        ("traces", Traces),
        ("profiles", c_void_p),
        ("n_profiles", c_int32),
        ("flags", c_int32),
        ("instances", c_void_p),
        ("n_instances", c_int64),
        ("summaries", c_void_p),
        ("rows", Rows),
        ("trace_buf", c_void_p),
        ("lut_out_sums", c_void_p),
        ("lut_out_counts", c_void_p),
        ("max_requests", c_int64),
        ("order", c_void_p),
        ("rows_capacity", c_int64),
        ("trace_buf_capacity", c_int64),
    ]


# numpy dtype of Summary (for zero-copy views of the summary array)
def summary_dtype():
    import numpy as np

    return np.dtype(
        [
            ("status", "<i4"), ("n", "<i4"), ("ttft_met", "<i4"), ("tpot_met", "<i4"),
            ("e2e_met", "<i4"), ("n_tps", "<i4"), ("tps_p50", "<f8"), ("tps_p90", "<f8"),
            ("worst_queue_wait_us", "<i8"), ("prefill_steps", "<i8"), ("decode_steps", "<i8"),
            ("digest", "<u8"), ("v_dec", "<i8"), ("b_dec", "<i8"), ("v_pre", "<i8"),
            ("deadline_misses", "<i8"), ("t_end_us", "<i8"), ("est_tokens", "<i8"),
            ("est_busy_us", "<i8"), ("max_queue", "<i4"), ("max_active", "<i4"), ("sim_cycles", "<i8"),
        ]
    )


def instance_dtype():
    import numpy as np

    return np.dtype(
        [
            ("trace_offset", "<i8"), ("n_requests", "<i4"), ("profile_id", "<i4"),
            ("rescale_factor", "<f8"), ("ttft_slo_us", "<i8"), ("tpot_slo_us", "<i8"),
            ("kv_capacity_tokens", "<i8"), ("transfer_base_us", "<i8"),
            ("transfer_per_token_us", "<f8"), ("chunk_budget", "<i4"), ("prefill_policy", "i1"),
            ("decode_policy", "i1"), ("_pad1", "i1", (2,)), ("rng_state_hi", "<u8"),
            ("rng_state_lo", "<u8"), ("rng_inc_hi", "<u8"), ("rng_inc_lo", "<u8"),
            ("row_offset", "<i8"), ("trace_buf_offset", "<i8"), ("trace_buf_words", "<i8"),
        ]
    )


assert ctypes.sizeof(Summary) == 144
assert ctypes.sizeof(Instance) == 128

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLOSIM_LIB") or os.path.join(_HERE, "libslosim_b200.so")
_lib = None


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or no CUDA device is present (no CPU fallback)."""


def lib():
    """Load the CUDA C-ABI library; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(LIB_PATH)
    vp = c_void_p
    L.slosim_run_batch.argtypes = [POINTER(Batch), vp]
    L.slosim_run_batch_host.argtypes = [POINTER(Batch), POINTER(c_float)]
    L.slosim_workspace_bytes.argtypes = [POINTER(Batch)]
    L.slosim_workspace_bytes.restype = c_int64
    L.slosim_synth_profile.argtypes = [POINTER(Profile), c_int32, vp, vp, vp, c_double, c_int64]
    L.slosim_lut_lookup.argtypes = [c_int32, vp, c_int32, vp, vp, vp, c_int64, vp, vp, vp]
    L.slosim_decode_formula.argtypes = [c_int32, vp, vp, c_double, c_int64, vp, vp, vp]
    L.slosim_estimate_duration.argtypes = [c_int64, c_int64, c_int64, vp, vp]
    L.slosim_predict_finish.argtypes = [c_int32, vp, vp, c_int64, c_int64, c_int64, vp]
    L.slosim_select_prefill.argtypes = [c_int32, c_int32, vp, vp, vp, vp, c_int64, c_int64, c_int64,
                                        c_int64, c_int64, vp, vp, vp, vp]
    L.slosim_select_decode.argtypes = [c_int32, c_int32, vp, vp, vp, vp, c_double, c_int64, c_int32, vp,
                                       c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.slosim_prefill_batch_us.argtypes = [c_int32, vp, vp, c_int32, vp, vp, vp]
    L.slosim_request_metrics.argtypes = [c_int64, vp, vp, vp, vp, c_int64, c_int64, vp, vp, vp, vp, vp, vp]
    L.slosim_histogram.argtypes = [c_int64, vp, vp, c_int32, vp, vp]
    L.slosim_exchange.argtypes = [vp, vp, c_int64, vp, vp, c_int64, vp]
    L.slosim_gen_longtail.argtypes = [vp, c_int64, vp, vp, vp, vp, vp, c_int64, vp, vp]
    L.slosim_gen_longtail_host.argtypes = [vp, c_int64, vp, vp, vp, vp, vp, c_int64, vp]
    L.slosim_rng_draws.argtypes = [c_int32, vp, c_int64, c_int64, c_double, c_double, vp, vp]
    L.slosim_libm.argtypes = [c_int32, c_int64, vp, vp, vp]
    L.slosim_abi_version.restype = c_int
    L.slosim_last_error.restype = c_char_p
    L.slosim_build_info.restype = c_char_p
    L.slosim_device_count.restype = c_int
    if L.slosim_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: the simulator has no CPU fallback")
    _lib = L
    return L


# exported C symbols that include/slosim_b200.h declares (checked by tests)
HEADER_SYMBOLS = [
    "slosim_last_error",
    "slosim_exchange",
    "slosim_run_batch",
    "slosim_run_batch_host",
    "slosim_workspace_bytes",
    "slosim_synth_profile",
    "slosim_lut_lookup",
    "slosim_decode_formula",
    "slosim_estimate_duration",
    "slosim_predict_finish",
    "slosim_select_prefill",
    "slosim_select_decode",
    "slosim_prefill_batch_us",
    "slosim_request_metrics",
    "slosim_histogram",
    "slosim_gen_longtail",
    "slosim_gen_longtail_host",
    "slosim_rng_draws",
    "slosim_libm",
    "slosim_abi_version",
    "slosim_device_count",
    "slosim_build_info",
]
