"""GPU: gen_longtail on the device (slosim_gen_longtail, csrc/rng.cuh) against numpy,
libm and the reference's own traces, bit for bit.

The oracle is the reference's dependency itself (numpy's Generator and the libm exp/log1p it calls,
both present on the GPU box) and the golden traces recorded from the unmodified reference
(tests/golden/make_longtail_golden.py).  tests/test_rng_host.py checks the same source on the CPU.
"""

import ctypes
import math

import numpy as np
import pytest

from test_rng_host import DRAWS, EDGE_SPECS, _libm_inputs, golden_specs, numpy_draws, trace_sha

pytestmark = pytest.mark.gpu


def L():
    from paper_2605_02329_b200 import _abi

    return _abi.lib()


def ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.mark.parametrize("fn", [0, 1], ids=["exp", "log1p"])
def test_device_libm_equals_host_libm(fn):
    xs = np.concatenate([_libm_inputs(fn), np.random.default_rng(fn).uniform(-1 if fn else -40, 40, 2_000_000)])
    y = np.zeros_like(xs)
    ok = np.zeros(len(xs), np.uint8)
    assert L().slosim_libm(fn, len(xs), ptr(xs), ptr(y), ptr(ok)) == 0
    f = math.exp if fn == 0 else math.log1p
    ref = np.array([f(v) for v in xs])
    assert ok.all()
    bad = np.flatnonzero(ref.view(np.uint64) != y.view(np.uint64))
    assert bad.size == 0, [(xs[i], ref[i], y[i]) for i in bad[:5]]


@pytest.mark.parametrize("kind,f,p0,p1", DRAWS, ids=[f"k{d[0]}_{i}" for i, d in enumerate(DRAWS)])
def test_device_draws_equal_numpy_1e7(kind, f, p0, p1):
    """>= 10^7 draws per Generator method (1,024 seeds x 10,000), every bit equal to numpy's."""
    seeds = np.arange(1024, dtype=np.uint64) * 7919 + 3
    n = 10_000
    got = np.zeros(len(seeds) * n, np.uint64)
    st = np.zeros(len(seeds), np.int32)
    assert L().slosim_rng_draws(kind, ptr(seeds), len(seeds), n, p0, p1, ptr(got), ptr(st)) == 0
    assert (st == 0).all()
    want = numpy_draws(kind, f, seeds, n)
    bad = np.argwhere(want != got.reshape(len(seeds), n))
    assert bad.size == 0, bad[:5]


def test_device_traces_equal_reference_golden():
    """All golden traces of the reference's gen_longtail: config 1's, config 2's 100k trace, 8 config-4
    seeds, all 256 config-5 seeds and the edge specs."""
    from paper_2605_02329_b200.workload import longtail_arrays_device

    full, hashed = golden_specs()
    for (spec, rows, _), tr in zip(full, longtail_arrays_device([f[0] for f in full])):
        got = np.stack([tr.arrival_us, tr.input_len, tr.output_len, tr.prefix_hit_len], axis=1)
        assert np.array_equal(got, rows), spec
    for (spec, sha, _), tr in zip(hashed, longtail_arrays_device([h[0] for h in hashed])):
        assert trace_sha(tr.arrival_us, tr.input_len, tr.output_len, tr.prefix_hit_len) == sha, spec


def test_device_traces_equal_host_generator_config4_and_edges():
    """Config 4's 256 traces of 20k requests (5.12M requests) and the edge specs vs numpy on the host."""
    from paper_2605_02329_b200.workload import LongTailSpec, longtail_arrays, longtail_arrays_device

    specs = EDGE_SPECS + [LongTailSpec(n_requests=20_000, seed=s, qps=4.0) for s in range(256)]
    for spec, tr in zip(specs, longtail_arrays_device(specs)):
        ref = longtail_arrays(spec)
        for k in ("arrival_us", "input_len", "output_len", "prefix_hit_len", "id_rank"):
            assert np.array_equal(getattr(tr, k), getattr(ref, k)), (spec, k)


def test_device_resident_generation_is_stream_ordered():
    """slosim_gen_longtail with device pointers on a side stream: same bytes as the host entry point;
    positions no spec covers are untouched; a rejected spec gets EINVAL and writes nothing."""
    import torch

    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200.workload import LongTailSpec, _spec_struct, longtail_arrays_device

    specs = [LongTailSpec(seed=s) for s in range(40)]
    bad = LongTailSpec(n_requests=10, seed=1)
    bad.p_long = 2.0
    offs = [k * 1100 for k in range(41)]  # 100-request gaps between traces
    structs = [_spec_struct(s, o) for s, o in zip(specs + [bad], offs)]
    arr = (_abi.LongTailSpec * len(structs))(*structs)
    n_total = offs[-1] + 10
    dev = torch.device("cuda:0")
    d_spec = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(dev)
    a = torch.full((n_total,), -5, dtype=torch.int64, device=dev)
    i32 = [torch.full((n_total,), -5, dtype=torch.int32, device=dev) for _ in range(4)]
    st = torch.full((len(structs),), -1, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rc = L().slosim_gen_longtail(d_spec.data_ptr(), len(structs), a.data_ptr(), *[t.data_ptr() for t in i32],
                                     n_total, st.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    assert rc == 0
    s.synchronize()
    st = st.cpu().numpy()
    assert (st[:-1] == 0).all() and st[-1] == _abi.EINVAL
    a = a.cpu().numpy()
    inp, out, hit, idr = (t.cpu().numpy() for t in i32)
    for k, tr in enumerate(longtail_arrays_device(specs)):
        sl = slice(offs[k], offs[k] + 1000)
        assert np.array_equal(a[sl], tr.arrival_us) and np.array_equal(inp[sl], tr.input_len)
        assert np.array_equal(out[sl], tr.output_len) and not hit[sl].any() and np.array_equal(idr[sl], tr.id_rank)
        gap = slice(offs[k] + 1000, offs[k + 1])
        assert (a[gap] == -5).all() and (inp[gap] == -5).all()


def test_config1_runs_identically_on_device_generated_traces():
    from paper_2605_02329_b200.batch import config1, run_batch

    host = run_batch(config1().packed).copy()
    dev = run_batch(config1(gen="device").packed).copy()
    for k in host.dtype.names:
        if k != "sim_cycles":
            assert np.array_equal(host[k], dev[k], equal_nan=host[k].dtype.kind == "f"), k
