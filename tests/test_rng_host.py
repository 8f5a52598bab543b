"""CPU: the device workload generator's source (csrc/rng.cuh) compiled as host C++ by the harness
tools/rng_host, against numpy and libm themselves (gen_longtail workload.py:88-112).

The oracle here is the reference's own dependency: numpy 2.3.5's Generator (default_rng ->
SeedSequence -> PCG64; exponential, random, lognormal, integers) and the libm exp/log1p it calls.
Every comparison is bit-for-bit.  tests/test_gpu_longtail.py runs the same checks on the device.
"""

import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.workload import LongTailSpec, longtail_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "tools", "rng_host")
P = ctypes.c_void_p


def ptr(a):
    return a.ctypes.data_as(P)


@pytest.fixture(scope="module")
def rh():
    subprocess.run(["bash", os.path.join(HARNESS, "build.sh")], check=True)
    return ctypes.CDLL(os.path.join(HARNESS, "librng_host.so"))


SEEDS = [0, 1, 2, 7, 2024, 12345, 2**31 - 1, 2**32 - 1, 2**32, 2**32 + 1, 2**40 + 5, 2**63, 2**64 - 1]


def test_seed_sequence_and_pcg64_state(rh):
    for seed in SEEDS + list(range(100, 300)):
        o = np.zeros(4, np.uint64)
        rh.rng_host_seed_state(ctypes.c_uint64(seed), ptr(o))
        st = np.random.default_rng(seed).bit_generator.state["state"]
        assert (int(o[0]) << 64 | int(o[1])) == int(st["state"]), seed
        assert (int(o[2]) << 64 | int(o[3])) == int(st["inc"]), seed


def _libm_inputs(fn):
    rs = np.random.default_rng(99)
    if fn == 0:  # exp: the draws' arguments (-x of the exponential wedge, -x^2/2, lognormal) and edges
        xs = [rs.uniform(-30, 30, 300_000), -rs.exponential(2.0, 200_000), -0.5 * rs.normal(0, 1.5, 200_000) ** 2,
              rs.normal(np.log(2048.0), 1.0, 200_000), rs.normal(np.log(150.0), 0.7, 200_000),
              np.array([0.0, -0.0, 1e-300, -1e-300, 2.0**-54, -(2.0**-55), 2.0**-53, 1.0, -1.0, 300.0, -300.0,
                        511.9, -511.9])]
    else:  # log1p: -U of the ziggurat tails, plus every branch of the fdlibm code
        edges = [0.0, -0.0, 2.0**-60, -(2.0**-60), 2.0**-30, -(2.0**-30), 2.0**-29, 0.41421, 0.41422, 0.4142136,
                 -0.29289, -0.2928932, -0.2929, -0.5, -0.9999999999999999, 1.0, 3.0, 1e10, 2.0**53, 2.0**60, 1e300]
        xs = [-rs.random(500_000), rs.uniform(-1, 4, 200_000), -rs.random(50_000) * 1e-6, rs.random(50_000) * 1e-6,
              -1 + rs.random(50_000) * 1e-9, rs.exponential(1e6, 50_000), np.array(edges)]
    return np.concatenate(xs)


@pytest.mark.parametrize("fn", [0, 1], ids=["exp", "log1p"])
def test_libm_restatement_equals_libm(rh, fn):
    xs = _libm_inputs(fn)
    y = np.zeros_like(xs)
    ok = np.zeros(len(xs), np.uint8)
    rh.rng_host_libm(fn, ctypes.c_int64(len(xs)), ptr(xs), ptr(y), ptr(ok))
    f = math.exp if fn == 0 else math.log1p
    ref = np.array([f(v) for v in xs])
    assert ok.all()
    bad = np.flatnonzero(ref.view(np.uint64) != y.view(np.uint64))
    assert bad.size == 0, [(xs[i], ref[i], y[i]) for i in bad[:5]]
    # outside the restated domain the call reports it instead of answering
    out = np.array([700.0, -800.0, np.inf, np.nan] if fn == 0 else [-1.0, -2.0, np.inf, np.nan])
    ok2 = np.ones(len(out), np.uint8)
    rh.rng_host_libm(fn, ctypes.c_int64(len(out)), ptr(out), ptr(np.zeros_like(out)), ptr(ok2))
    assert not ok2.any()


DRAWS = [
    (_abi.DRAW_RAW, lambda g, n: g.bit_generator.random_raw(n).astype(np.uint64), 0.0, 0.0),
    (_abi.DRAW_RANDOM, lambda g, n: g.random(n), 0.0, 0.0),
    (_abi.DRAW_STD_EXPONENTIAL, lambda g, n: g.standard_exponential(n), 0.0, 0.0),
    (_abi.DRAW_EXPONENTIAL, lambda g, n: g.exponential(1.0 / 3.7, n), 1.0 / 3.7, 0.0),
    (_abi.DRAW_STD_NORMAL, lambda g, n: g.standard_normal(n), 0.0, 0.0),
    (_abi.DRAW_LOGNORMAL, lambda g, n: g.lognormal(math.log(2048.0), 1.0, n), math.log(2048.0), 1.0),
    (_abi.DRAW_LOGNORMAL, lambda g, n: g.lognormal(math.log(150.0), 0.7, n), math.log(150.0), 0.7),
    (_abi.DRAW_INTEGERS, lambda g, n: g.integers(65536, 131073, n), 65536.0, 131073.0),
    (_abi.DRAW_INTEGERS, lambda g, n: g.integers(0, 2**32 - 1, n), 0.0, 2.0**32 - 1),
    (_abi.DRAW_INTEGERS, lambda g, n: g.integers(5, 12, n), 5.0, 12.0),
]


def numpy_draws(kind, f, seeds, n):
    out = np.zeros((len(seeds), n), np.uint64)
    for i, s in enumerate(seeds):
        r = np.asarray(f(np.random.default_rng(int(s)), n))
        out[i] = r.view(np.uint64) if r.dtype == np.float64 else r.astype(np.int64).view(np.uint64)
    return out


@pytest.mark.parametrize("kind,f,p0,p1", DRAWS, ids=[f"k{d[0]}_{i}" for i, d in enumerate(DRAWS)])
def test_draws_equal_numpy(rh, kind, f, p0, p1):
    seeds = np.array(SEEDS + list(range(1000, 1128)), np.uint64)
    n = 8000  # ~1.1M draws per method: thousands of ziggurat wedge and tail draws
    got = np.zeros(len(seeds) * n, np.uint64)
    st = np.zeros(len(seeds), np.int32)
    rh.rng_host_draws(kind, ptr(seeds), ctypes.c_int64(len(seeds)), ctypes.c_int64(n), ctypes.c_double(p0),
                      ctypes.c_double(p1), ptr(got), ptr(st))
    assert (st == 0).all()
    want = numpy_draws(kind, f, seeds, n)
    bad = np.argwhere(want != got.reshape(len(seeds), n))
    assert bad.size == 0, bad[:5]


def host_gen(rh, specs):
    from paper_2605_02329_b200.workload import _spec_struct

    n = [s.n_requests for s in specs]
    offs = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64) if specs else np.zeros(0, np.int64)
    total = int(sum(n))
    arr = (_abi.LongTailSpec * len(specs))(*[_spec_struct(s, o) for s, o in zip(specs, offs)])
    a = np.zeros(max(total, 1), np.int64)
    inp, out, hit, idr = (np.full(max(total, 1), 7, np.int32) for _ in range(4))
    st = np.zeros(len(specs), np.int32)
    rh.rng_host_gen_longtail(arr, ctypes.c_int64(len(specs)), ptr(a), ptr(inp), ptr(out), ptr(hit), ptr(idr),
                             ctypes.c_int64(total), ptr(st))
    return [(st[i], a[o:o + k], inp[o:o + k], out[o:o + k], hit[o:o + k], idr[o:o + k])
            for i, (o, k) in enumerate(zip(offs, n))]


EDGE_SPECS = [
    LongTailSpec(),  # config 1 / 3
    LongTailSpec(n_requests=100_000, seed=2024, qps=1.0),  # config 2
    LongTailSpec(n_requests=20_000, seed=3, qps=4.0),  # config 4
    LongTailSpec(n_requests=0),
    LongTailSpec(n_requests=1, seed=5),
    LongTailSpec(n_requests=500, p_long=1.0, seed=6),
    LongTailSpec(n_requests=500, p_long=0.0, seed=7),
    LongTailSpec(n_requests=500, short_len_log_sigma=0.0, out_len_log_sigma=0.0, seed=8),
    LongTailSpec(n_requests=500, long_len_min=7, long_len_max=7, p_long=0.5, seed=9),
    LongTailSpec(n_requests=2000, qps=250.0, seed=2**40 + 3),
    LongTailSpec(n_requests=2000, qps=0.01, out_len_log_sigma=2.5, short_len_log_sigma=2.0, seed=11),
    LongTailSpec(n_requests=300, long_len_min=1, long_len_max=2**31 - 2, p_long=0.3, seed=12),
]


def test_traces_equal_reference_generator(rh):
    specs = EDGE_SPECS + [LongTailSpec(seed=s) for s in range(64)]
    for spec, (st, a, inp, out, hit, idr) in zip(specs, host_gen(rh, specs)):
        tr = longtail_arrays(spec)
        assert st == _abi.OK
        assert np.array_equal(a, tr.arrival_us), spec
        assert np.array_equal(inp, tr.input_len), spec
        assert np.array_equal(out, tr.output_len), spec
        assert not hit.any() and np.array_equal(idr, np.arange(len(a))), spec


def golden_specs():
    """Specs and expected traces recorded from the unmodified reference (tests/golden/make_longtail_golden.py)."""
    from helpers import load_golden

    g = load_golden("longtail_golden.json.gz")
    full = [(LongTailSpec(**e["spec"]), np.array(e["rows"], np.int64).reshape(-1, 4), e["ids"]) for e in g["full"]]
    hashed = [(LongTailSpec(**e["spec"]), e["sha256"], e["ids_in_position_order"]) for e in g["sha256"]]
    return full, hashed


def trace_sha(a, inp, out, hit):
    import hashlib

    cols = np.stack([a, inp.astype(np.int64), out.astype(np.int64), hit.astype(np.int64)], axis=1)
    return hashlib.sha256(np.ascontiguousarray(cols).tobytes()).hexdigest()


def test_traces_equal_reference_golden(rh):
    """Every golden trace of the reference's gen_longtail: 6 in full (ids in position order), 265 by hash
    (config 2's 100k trace, 8 config-4 seeds, all 256 config-5 seeds)."""
    full, hashed = golden_specs()
    for (spec, rows, ids), (st, a, inp, out, hit, idr) in zip(full, host_gen(rh, [f[0] for f in full])):
        assert st == _abi.OK
        w = max(4, len(str(max(spec.n_requests, 1))))
        assert ids == [f"r{k:0{w}d}" for k in range(len(ids))]
        assert np.array_equal(np.stack([a, inp, out, hit], axis=1), rows), spec
    for (spec, sha, in_order), (st, a, inp, out, hit, idr) in zip(hashed, host_gen(rh, [h[0] for h in hashed])):
        assert st == _abi.OK and in_order
        assert trace_sha(a, inp, out, hit) == sha, spec


def test_invalid_specs_rejected(rh):
    bad = [LongTailSpec(n_requests=10, seed=1), LongTailSpec(n_requests=10, seed=2)]
    bad[0].qps = -1.0  # bypass __post_init__: the C-ABI checks again
    bad[1].p_long = 1.5
    res = host_gen(rh, bad)
    assert [r[0] for r in res] == [_abi.EINVAL, _abi.EINVAL]
