"""GPU: the C-ABI contract of slosim_run_batch (include/slosim_b200.h) and the
multi-rank paths of the benchmark and the exchange.

- a malformed instance descriptor gets summary status SLOSIM_EINVAL and leaves every other
  instance's results untouched (no out-of-bounds writes into neighbouring workspaces);
- two batches enqueued on two concurrent streams give the results of sequential calls;
- the latency build and the throughput build of the engine give identical summaries and rows;
- `bench.py --gpus 2` runs two real ranks (gloo, sharing this GPU) whose exchanged histogram and
  gathered rows equal a one-rank run over the same slices;
- slosim_exchange over an ncclCommInitAll communicator of every visible GPU (skipped below 2).
"""

import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fields(a):
    return [x for x in a.dtype.names if x != "sim_cycles"]


def _same(a, b):
    for k in _fields(a):
        x, y = a[k], b[k]
        ok = np.array_equal(x, y, equal_nan=True) if x.dtype.kind == "f" else np.array_equal(x, y)
        if not ok:
            return k
    return None


def test_malformed_descriptors_get_einval_and_touch_nothing_else():
    import torch

    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200.batch import DeviceBatch, config3

    sw = config3(select=np.arange(64))
    db = DeviceBatch(sw.packed)
    db.launch()
    want = db.fetch().copy()

    inst = sw.packed.instances.copy()
    n_total = len(sw.packed.arrival)
    bad = {3: ("n_requests", 5000),            # beyond max_requests (1000): would overflow the workspace
           9: ("profile_id", 7),               # only one profile
           17: ("trace_offset", n_total - 10),  # trace range past the end of the trace table
           21: ("decode_policy", 5),
           30: ("chunk_budget", 0),
           41: ("trace_offset", -4)}
    for i, (f, v) in bad.items():
        inst[i][f] = v
    sw.packed.instances = inst
    db2 = DeviceBatch(sw.packed)
    db2.struct.max_requests = 1000
    db2.launch()
    got = db2.fetch().copy()
    for i in range(len(inst)):
        if i in bad:
            assert got[i]["status"] == _abi.EINVAL, (i, bad[i], got[i]["status"])
        else:
            assert _same(got[i:i + 1], want[i:i + 1]) is None, i
    torch.cuda.synchronize()


def test_order_entries_out_of_range_are_skipped():
    import torch

    from paper_2605_02329_b200.batch import DeviceBatch, config1

    sw = config1()
    db = DeviceBatch(sw.packed)
    db.launch()
    want = db.fetch().copy()
    order = np.array([0, 99, 1, -3, 2, 3, 4, 5, 6, 7, 8, 9], np.int64)  # 10, 11 absent; two junk entries
    db2 = DeviceBatch(sw.packed, order=order)
    db2.summaries.fill_(0)
    db2.launch()
    got = db2.fetch().copy()
    for i in range(10):
        assert _same(got[i:i + 1], want[i:i + 1]) is None, i
    assert got[10]["n"] == 0 and got[11]["n"] == 0  # never simulated
    torch.cuda.synchronize()


def test_concurrent_streams_give_sequential_results():
    import torch

    from paper_2605_02329_b200.batch import DeviceBatch, config3

    a = DeviceBatch(config3(select=np.arange(0, 600)).packed)
    b = DeviceBatch(config3(select=np.arange(600, 1400)).packed)
    a.launch()
    want_a = a.fetch().copy()
    b.launch()
    want_b = b.fetch().copy()
    for _ in range(3):
        a.summaries.zero_()
        b.summaries.zero_()
        torch.cuda.synchronize()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        a.launch(stream=s1)
        b.launch(stream=s2)
        torch.cuda.synchronize()
        assert _same(a.fetch(), want_a) is None
        assert _same(b.fetch(), want_b) is None


@pytest.mark.parametrize("env", ["SLOSIM_FORCE_LATENCY_ENGINE", "SLOSIM_NO_LATENCY_ENGINE"])
def test_latency_and_throughput_builds_agree(env, monkeypatch):
    """The same batch through both engine builds (spill-free latency build and the throughput build):
    summaries and per-request rows identical, and both equal the golden reference outputs."""
    from helpers import load_golden, pack_cases, row_mismatches, summary_mismatches

    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200.batch import run_batch

    cases = load_golden()["cases"][:120] + load_golden("extra_golden.json.gz")[:24]
    monkeypatch.setenv(env, "1")
    packed, _ = pack_cases(cases, flags=_abi.F_ROWS)
    got = run_batch(packed)
    bad = {}
    for i, c in enumerate(cases):
        m = summary_mismatches(got[i], c["summary"])
        if c["summary"]["status"] == 0:
            m += row_mismatches(packed, i, c["summary"]["rows"])[:3]
        if m:
            bad[i] = m
    assert not bad, f"{env}: {len(bad)} cases differ: {dict(list(bad.items())[:4])}"


def _bench(args, env_extra=None, timeout=900):
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env, capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(1200)
def test_bench_two_ranks_equal_one_rank():
    """bench.py --gpus 2 spawns two ranks itself (gloo, both on this GPU); rank r takes slices s*2+r.
    Timed slices {2, 3} on two ranks (1 step each) equal timed slices {2, 3} on one rank (2 steps):
    the all-reduced histogram and the all-gathered summary rows must be identical."""
    common = ["--slice", "256", "--no-e2e", "--no-cpu"]
    two = _bench(["--gpus", "2", "--steps", "1", "--warmup", "1"] + common, {"SLOSIM_DIST_BACKEND": "gloo"})
    one = _bench(["--gpus", "1", "--steps", "2", "--warmup", "2"] + common)
    assert two["n_gpus"] == 2 and two["exchange"]["ranks"] == 2
    assert one["n_gpus"] == 1
    for line in (one, two):
        ex = line["exchange"]
        assert ex["rows_gathered"] == ex["rows_expected"] == 512
        assert ex["hist_total"] == 512
        assert ex["own_rows_in_place"]
    assert two["exchange"]["hist_sha16"] == one["exchange"]["hist_sha16"]
    assert two["exchange"]["rows_sha16"] == one["exchange"]["rows_sha16"]


def test_exchange_over_nccl_all_visible_devices():
    """Single-process multi-GPU mode: one communicator per device from
    ncclCommInitAll, each device runs its shard, then slosim_exchange in one NCCL group."""
    import torch

    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200 import dist as D
    from paper_2605_02329_b200.batch import DeviceBatch, config3

    G = torch.cuda.device_count()
    if G < 2:
        pytest.skip(f"{G} GPU visible; the N-rank exchange needs >= 2")
    L = _abi.lib()
    n_per = 64
    idx = [np.arange(r, G * n_per, G) for r in range(G)]  # strided shards
    full = config3(select=np.arange(G * n_per))
    cells_all = D.cell_ids_config_grid(np.arange(G * n_per), 3, 16, 64)
    full_summ = _run_on(0, full.packed)
    want = D.host_histogram(full_summ, cells_all, 3 * 16 * 64, 1001)
    nccl = ctypes.CDLL("libnccl.so.2")
    comms = (ctypes.c_void_p * G)()
    devs = (ctypes.c_int * G)(*range(G))
    assert nccl.ncclCommInitAll(comms, G, devs) == 0
    outs, hists, mines = [], [], []
    try:
        for r in range(G):
            with torch.cuda.device(r):
                sw = config3(select=idx[r])
                db = DeviceBatch(sw.packed, device=f"cuda:{r}")
                db.launch()
                cells = torch.from_numpy(D.cell_ids_config_grid(idx[r], 3, 16, 64)).to(f"cuda:{r}")
                h = torch.zeros(3 * 16 * 64 * 1001, dtype=torch.int64, device=f"cuda:{r}")
                st = torch.cuda.current_stream(r)
                assert L.slosim_histogram(n_per, ctypes.c_void_p(db.summaries.data_ptr()),
                                          ctypes.c_void_p(cells.data_ptr()), 1001, ctypes.c_void_p(h.data_ptr()),
                                          ctypes.c_void_p(st.cuda_stream)) == 0
                mines.append(db)
                hists.append(h)
                outs.append(torch.zeros(G * n_per * 144, dtype=torch.uint8, device=f"cuda:{r}"))
        assert nccl.ncclGroupStart() == 0
        for r in range(G):
            with torch.cuda.device(r):
                st = torch.cuda.current_stream(r)
                rc = L.slosim_exchange(ctypes.c_void_p(comms[r]), ctypes.c_void_p(mines[r].summaries.data_ptr()),
                                       n_per, ctypes.c_void_p(outs[r].data_ptr()), ctypes.c_void_p(hists[r].data_ptr()),
                                       hists[r].numel(), ctypes.c_void_p(st.cuda_stream))
                assert rc == 0, L.slosim_last_error()
        assert nccl.ncclGroupEnd() == 0
        for r in range(G):
            torch.cuda.synchronize(r)
    finally:
        for r in range(G):
            nccl.ncclCommDestroy(ctypes.c_void_p(comms[r]))
    for r in range(G):
        assert np.array_equal(hists[r].cpu().numpy().reshape(want.shape), want)
        rows = D.summaries_from_bytes(outs[r])
        assert sorted(int(x) for x in rows["digest"]) == sorted(int(x) for x in full_summ["digest"])


def _run_on(dev, packed):
    from paper_2605_02329_b200.batch import DeviceBatch

    db = DeviceBatch(packed, device=f"cuda:{dev}")
    db.launch()
    return db.fetch().copy()
