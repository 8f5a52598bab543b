"""Multi-GPU sharding and the final exchange (K6 of SURVEY §2, §8(e)).

Instances are independent, so the path shards with no data-path collective:
rank r of G simulates the instance slices ``s*G + r``; every rank therefore
gets the same mix of rates / SLO scales / policies (strided assignment).  The
only exchange is at the end: an integer all-reduce of the per-(pair, rate,
SLO) e2e-attainment histograms and an all-gather of the fixed-size summary
rows.  Integer sums are order-independent, so the result is bit-exact for
any G.  Backend: NCCL over NVLink on GPUs; gloo in the CPU tests.
"""

from __future__ import annotations

import numpy as np

from . import _abi

SUMMARY_BYTES = 144


def slices_for_rank(n_slices: int, world: int, rank: int, steps: int, first_step: int = 0) -> list:
    """Slice ids processed by `rank` at steps first_step .. first_step+steps-1 (weak scaling)."""
    return [((first_step + s) * world + rank) % n_slices for s in range(steps)]


def cell_ids_config_grid(idx: np.ndarray, n_pairs: int, n_slo: int, n_rates: int) -> np.ndarray:
    """(pair, rate, slo) histogram cell of each grid instance index (batch.grid_batch decomposition)."""
    p = idx % n_pairs
    s = (idx // n_pairs) % n_slo
    r = (idx // (n_pairs * n_slo)) % n_rates
    return ((p * n_rates + r) * n_slo + s).astype(np.int32)


def host_histogram(summaries: np.ndarray, cells: np.ndarray, n_cells: int, n_bins: int) -> np.ndarray:
    """Reference histogram on the host (tests)."""
    h = np.zeros((n_cells, n_bins), np.int64)
    e = np.clip(summaries["e2e_met"].astype(np.int64), 0, n_bins - 1)
    np.add.at(h, (cells.astype(np.int64), e), 1)
    return h


def exchange(summary_bytes, hist, group=None):
    """Final exchange: all-reduce(sum, int64) of `hist`, all-gather of `summary_bytes`.

    `summary_bytes` is a uint8 tensor of this rank's summary rows (same length
    on every rank); `hist` an int64 tensor.  Returns (gathered uint8 tensor
    [world * n], hist reduced in place).  Works for any torch.distributed
    backend; with no initialised process group it is the identity.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return summary_bytes, hist
    world = dist.get_world_size(group)
    dev = hist.device
    if dist.get_backend(group) != "nccl" and dev.type == "cuda":  # gloo: exchange through host copies
        summary_bytes, hist = summary_bytes.cpu(), hist.cpu()
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    out = torch.empty(world * summary_bytes.numel(), dtype=summary_bytes.dtype, device=summary_bytes.device)
    dist.all_gather_into_tensor(out, summary_bytes, group=group)
    return out.to(dev), hist.to(dev)


def summaries_from_bytes(buf) -> np.ndarray:
    a = buf.detach().cpu().numpy() if hasattr(buf, "detach") else np.asarray(buf)
    return a.view(np.uint8).view(_abi.summary_dtype())
