"""CPU: host-side input packing (traces, rescale, sweep grids, histogram cells)."""

import numpy as np

from paper_2605_02329_b200 import dist as D
from paper_2605_02329_b200.batch import SWEEP_RATES, SWEEP_SLO_SCALES, config3
from paper_2605_02329_b200.domain import Request
from paper_2605_02329_b200.workload import (LongTailSpec, longtail_arrays, rescale_factor, rescale_qps,
                                            trace_arrays_from_requests)


def test_config1_trace_matches_appendix_c():
    """n=1000, first id r0000, last arrival 986,831,481, Σinput 8,246,030, Σoutput 195,128."""
    tr = longtail_arrays(LongTailSpec())
    assert len(tr) == 1000 and tr.id_of(0) == "r0000"
    assert int(tr.arrival_us[-1]) == 986_831_481
    assert int(tr.input_len.astype(np.int64).sum()) == 8_246_030
    assert int(tr.output_len.astype(np.int64).sum()) == 195_128
    assert int((tr.input_len >= 65536).sum()) == 53


def test_device_rescale_formula_equals_rescale_qps():
    tr = longtail_arrays(LongTailSpec(n_requests=300, seed=9))
    reqs = tr.to_requests()
    for q in (0.1, 0.7, 1.9, 3.25):
        f = rescale_factor(tr.arrival_us, q)
        dev = np.rint(tr.arrival_us.astype(np.float64) * f).astype(np.int64)
        assert dev.tolist() == [r.arrival_time for r in rescale_qps(reqs, q)]


def test_trace_packing_orders_by_arrival_then_id():
    wl = [Request("b", 0, 10, 1), Request("a", 0, 20, 2), Request("c", 5, 30, 3)]
    tr = trace_arrays_from_requests(wl)
    assert [tr.id_of(p) for p in range(3)] == ["a", "b", "c"]
    assert tr.id_rank.tolist() == [0, 1, 2]
    assert tr.input_len.tolist() == [20, 10, 30]


def test_grid_decomposition_and_cells():
    sw = config3(select=np.arange(0, 3072, 97), synth=_fake_synth)
    c = sw.coords
    idx = np.arange(0, 3072, 97)
    assert (c["pair"] == idx % 3).all()
    assert np.allclose(c["slo_scale"], np.array(SWEEP_SLO_SCALES)[(idx // 3) % 16])
    assert np.allclose(c["rate"], np.array(SWEEP_RATES)[(idx // 48) % 64])
    inst = sw.packed.instances
    assert (inst["ttft_slo_us"] == np.round(8e6 * c["slo_scale"]).astype(np.int64)).all()
    cells = D.cell_ids_config_grid(idx, 3, 16, 64)
    assert cells.max() < 3 * 16 * 64 and len(set(cells.tolist())) == len(idx)


def test_slices_for_rank_partition_steps():
    world, n_slices, steps = 4, 64, 16
    seen = [s for r in range(world) for s in D.slices_for_rank(n_slices, world, r, steps)]
    assert sorted(seen) == list(range(n_slices))


def _fake_synth(P, anchors, gamma, weight):
    """Packing-only tests do not need the LUT values."""
    P.lut_counts[0] = 1
    P.lut_sums[0] = 1.0
