"""CPU: the N>1 exchange (histogram all-reduce + summary all-gather) on a world_size-2 gloo group.

Each rank simulates its strided slices with the C oracle standing in for the
GPU engine; the exchanged histogram must equal the single-process histogram of
all instances, bit for bit (integer sums are order independent).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2605_02329_b200 import dist as D
    from paper_2605_02329_b200.batch import config3

    n_slices, slice_n = 8, 12
    mine = D.slices_for_rank(n_slices, world, rank, n_slices // world)
    idx = np.concatenate([np.arange(s * slice_n, (s + 1) * slice_n) for s in mine])
    sw = config3(select=idx, synth=oracle.synth)
    oracle.run_batch(sw.packed, threads=2)
    cells = D.cell_ids_config_grid(idx, 3, 16, 64)
    hist = torch.from_numpy(D.host_histogram(sw.packed.summaries, cells, 3 * 16 * 64, 1001).reshape(-1))
    summ = torch.from_numpy(sw.packed.summaries.view(np.uint8).copy())
    gathered, hist = D.exchange(summ, hist)
    if rank == 0:
        np.save(os.path.join(out_dir, "hist.npy"), hist.numpy())
        np.save(os.path.join(out_dir, "gathered.npy"), gathered.numpy())
        np.save(os.path.join(out_dir, "idx0.npy"), idx)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_exchange_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle import oracle
    from paper_2605_02329_b200 import dist as D
    from paper_2605_02329_b200.batch import config3

    allidx = np.arange(8 * 12)
    sw = config3(select=allidx, synth=oracle.synth)
    oracle.run_batch(sw.packed, threads=2)
    want = D.host_histogram(sw.packed.summaries, D.cell_ids_config_grid(allidx, 3, 16, 64), 3 * 16 * 64, 1001)
    got = np.load(tmp_path / "hist.npy").reshape(want.shape)
    assert np.array_equal(got, want)
    gathered = D.summaries_from_bytes(np.load(tmp_path / "gathered.npy"))
    assert len(gathered) == len(allidx)
    # every instance's summary row arrives exactly once
    by_digest = sorted(int(x) for x in gathered["digest"])
    assert by_digest == sorted(int(x) for x in sw.packed.summaries["digest"])
