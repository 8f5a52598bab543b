"""CPU: the C-ABI library exports every symbol include/slosim_b200.h declares, and the
ctypes mirror matches the C struct layouts (probe compiled with gcc)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2605_02329_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slosim_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(slosim_\w+)\s*\(", text, re.M)))


def test_header_symbol_list_matches_mirror():
    assert header_functions() == sorted(_abi.HEADER_SYMBOLS)


def test_library_exports_all_header_symbols():
    if not os.path.exists(_abi.LIB_PATH):
        from paper_2605_02329_b200 import _build

        _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (slosim_\w+)", out))
    missing = [s for s in header_functions() if s not in exported]
    assert not missing, missing
    # loading needs no GPU; calling compute does
    lib = ctypes.CDLL(_abi.LIB_PATH)
    lib.slosim_abi_version.restype = ctypes.c_int
    assert lib.slosim_abi_version() == 2


def test_lib_fails_loudly_without_device():
    """No CPU fallback: with no visible CUDA device the loader raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_abi.NativeUnavailable):
        _abi._lib = None
        _abi.lib()


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "slosim_b200.h"
#define P(T, f) printf("%s.%s %zu\n", #T, #f, offsetof(T, f));
int main(void) {
  printf("sizeof.profile %zu\nsizeof.instance %zu\nsizeof.summary %zu\nsizeof.batch %zu\nsizeof.rows %zu\n",
         sizeof(slosim_profile_t), sizeof(slosim_instance_t), sizeof(slosim_summary_t), sizeof(slosim_batch_t),
         sizeof(slosim_rows_t));
  P(slosim_profile_t, est_tokens) P(slosim_profile_t, curve_x) P(slosim_profile_t, base_y) P(slosim_profile_t, gamma)
  P(slosim_profile_t, gt_sums) P(slosim_profile_t, gt_counts)
  P(slosim_instance_t, rescale_factor) P(slosim_instance_t, chunk_budget) P(slosim_instance_t, rng_state_hi)
  P(slosim_instance_t, row_offset) P(slosim_instance_t, trace_buf_words)
  P(slosim_summary_t, tps_p50) P(slosim_summary_t, digest) P(slosim_summary_t, max_active)
  P(slosim_batch_t, profiles) P(slosim_batch_t, instances) P(slosim_batch_t, rows) P(slosim_batch_t, max_requests)
  P(slosim_batch_t, order) P(slosim_batch_t, rows_capacity) P(slosim_batch_t, trace_buf_capacity)
  P(slosim_longtail_spec_t, p_long) P(slosim_longtail_spec_t, seed) P(slosim_longtail_spec_t, offset)
  printf("sizeof.longtail %zu\n", sizeof(slosim_longtail_spec_t));
  return 0;
}
"""


def test_struct_layouts_match_ctypes(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(PROBE)
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    vals = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    m = {"profile": _abi.Profile, "instance": _abi.Instance, "summary": _abi.Summary, "batch": _abi.Batch,
         "rows": _abi.Rows, "longtail": _abi.LongTailSpec}
    for k, cls in m.items():
        assert int(vals[f"sizeof.{k}"]) == ctypes.sizeof(cls), k
    names = {"slosim_profile_t": _abi.Profile, "slosim_instance_t": _abi.Instance, "slosim_summary_t": _abi.Summary,
             "slosim_batch_t": _abi.Batch, "slosim_longtail_spec_t": _abi.LongTailSpec}
    for key, v in vals.items():
        if key.startswith("sizeof"):
            continue
        t, f = key.split(".")
        assert getattr(names[t], f).offset == int(v), key
    assert _abi.summary_dtype().itemsize == ctypes.sizeof(_abi.Summary)
    assert _abi.instance_dtype().itemsize == ctypes.sizeof(_abi.Instance)
