"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE — not the product).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It runs oracle/libslosim_oracle.so, a
plain-C restatement of the reference slosim engine (see slosim_oracle.c), on
the same packed batch the CUDA library consumes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libslosim_oracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        deps = [os.path.join(HERE, "slosim_oracle.c"), os.path.join(HERE, "..", "include", "slosim_b200.h")]
        if not os.path.exists(LIB) or any(os.path.getmtime(LIB) < os.path.getmtime(d) for d in deps):
            build()
        L = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.oracle_run_batch.argtypes = [vp, ctypes.c_int]
        L.oracle_lut_lookup.argtypes = [i32, vp, i32, vp, vp, vp, i64, vp, vp, vp]
        L.oracle_decode_formula.argtypes = [i32, vp, vp, f64, i64, vp, vp, vp]
        L.oracle_prefill_batch_us.argtypes = [i32, vp, vp, i32, vp, vp, vp]
        L.oracle_select_decode.argtypes = [i32, i32, vp, vp, vp, vp, f64, i64, i32, vp, i32, vp, vp, vp, vp, vp,
                                           vp, vp, vp, vp, vp, vp]
        L.oracle_select_prefill.argtypes = [i32, i32, vp, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp]
        L.oracle_predict_finish.argtypes = [i32, vp, vp, i64, i64, i64, vp]
        L.oracle_estimate_duration.argtypes = [i64, i64, i64, vp, vp]
        L.oracle_idiv.argtypes = [i64, i64]
        L.oracle_idiv.restype = f64
        L.oracle_synth_profile.argtypes = [vp, i32, vp, vp, vp, f64, i64]
        L.oracle_pcg_next.argtypes = [vp]
        L.oracle_pcg_next.restype = ctypes.c_uint64
        _lib = L
    return _lib


def synth(P, anchors, gamma, weight):
    """Oracle replacement of the device synth for packing batches on CPU-only hosts."""
    ab = np.array([int(a[0]) for a in anchors], np.int64)
    asq = np.array([int(a[1]) for a in anchors], np.int64)
    au = np.array([float(a[2]) for a in anchors], np.float64)
    rc = lib().oracle_synth_profile(ctypes.addressof(P), len(anchors), ab.ctypes.data, asq.ctypes.data,
                                    au.ctypes.data, float(gamma), int(weight))
    if rc:
        raise ValueError("synth failed")


def run_batch(packed, threads: int = 1):
    """Run every instance of a PackedBatch on the CPU oracle; fills packed.summaries/rows/trace_buf."""
    b = packed.host_struct()
    lib().oracle_run_batch(ctypes.addressof(b), int(threads))
    return packed


def lut_lookup(bsz_buckets, seq_buckets, sums, counts, bsz, seq):
    bb = np.asarray(bsz_buckets, np.int32); sb = np.asarray(seq_buckets, np.int32)
    s = np.ascontiguousarray(sums, np.float64); c = np.ascontiguousarray(counts, np.int32)
    qb = np.asarray(bsz, np.int64); qs = np.asarray(seq, np.int64)
    out = np.zeros(len(qb), np.float64)
    rc = lib().oracle_lut_lookup(len(bb), bb.ctypes.data, len(sb), sb.ctypes.data, s.ctypes.data, c.ctypes.data,
                                 len(qb), qb.ctypes.data, qs.ctypes.data, out.ctypes.data)
    assert rc == 0
    return out
