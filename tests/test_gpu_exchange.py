"""C-ABI multi-GPU exchange (slosim_exchange) over a real NCCL communicator.

One GPU per box here, so the communicator has one rank: the all-gather must copy
this rank's summary rows and the all-reduce must leave the histogram unchanged,
i.e. agree with dist.exchange's single-rank identity.  The multi-rank path is
the same two NCCL calls (tests/test_dist_gloo.py checks the merge logic with
world size 2)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_exchange_over_nccl_single_rank():
    import torch

    from paper_2605_02329_b200 import _abi
    from paper_2605_02329_b200 import dist as D
    from paper_2605_02329_b200.batch import DeviceBatch, config1

    sw = config1()
    db = DeviceBatch(sw.packed)
    db.launch()
    torch.cuda.synchronize()
    n = sw.packed.n_instances
    cells = torch.from_numpy(D.cell_ids_config_grid(np.arange(n), 2, 1, 6)).cuda()
    hist = torch.zeros(12 * 1001, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    L = _abi.lib()
    assert L.slosim_histogram(n, ctypes.c_void_p(db.summaries.data_ptr()), ctypes.c_void_p(cells.data_ptr()), 1001,
                              ctypes.c_void_p(hist.data_ptr()), ctypes.c_void_p(stream.cuda_stream)) == 0
    before = hist.clone()

    nccl = ctypes.CDLL("libnccl.so.2")
    comm = ctypes.c_void_p()
    dev = (ctypes.c_int * 1)(torch.cuda.current_device())
    assert nccl.ncclCommInitAll(ctypes.byref(comm), 1, dev) == 0
    try:
        out = torch.zeros_like(db.summaries)
        rc = L.slosim_exchange(comm, ctypes.c_void_p(db.summaries.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(hist.data_ptr()), hist.numel(), ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, L.slosim_last_error()
        torch.cuda.synchronize()
    finally:
        nccl.ncclCommDestroy(comm)
    assert torch.equal(out, db.summaries)
    assert torch.equal(hist, before)
    assert int(hist.sum()) == n
