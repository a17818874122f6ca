"""Host-side helpers for one-process-per-GPU runs (torch.distributed plumbing only).

Nothing here computes any part of the method: it decides which vertex rows a
rank owns (via the library's own ntp_partition), materialises that rank's slice
of the seeded synthetic inputs, bootstraps the library's NCCL communicator id
and reduces timings across ranks.
"""
from __future__ import annotations

import numpy as np


def rank_rows(n: int, w: int, world: int, rank: int, dtype: int = 0, slice_align: int = 16, slices: int = 0):
    """(row0, rows, V_p, d_s) of `rank`: rows [row0, row0+rows) are real vertices; V_p-rows is padding.
    slices = P feature slices (ntp_set_slices; default world): the rank owns V_pad / world rows."""
    from . import ntp
    P = slices or world
    part = ntp.partition(n, w, P, dtype, 1, slice_align)
    V_p = part["V_pad"] // world
    row0 = rank * V_p
    rows = max(0, min(V_p, n - row0))
    return row0, rows, V_p, part["d_s"]


def rank_inputs(cfg, world: int, rank: int, slices: int = 0):
    """This rank's VERTEX-layout inputs (X_v [V_p x d_in] fp32, labels int32, train mask uint8),
    zero-padded beyond n (padding rows are in no mask)."""
    import synth
    row0, rows, V_p, _ = rank_rows(cfg.n, cfg.w, world, rank, slices=slices)
    X = np.zeros((V_p, cfg.d_in), np.float32)
    y = np.zeros(V_p, np.int32)
    m = np.zeros(V_p, np.uint8)
    if rows:
        X[:rows], y[:rows], m[:rows] = synth.config_inputs(cfg, row0, rows)
    return X, y, m


def broadcast_unique_id(dist, rank: int):
    """Rank 0 creates the library's NCCL id; every rank receives the same 128 bytes."""
    from . import ntp
    obj = [ntp.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, value: float, device=None) -> float:
    """Max of a per-rank timing (the whole-job time of a step is the slowest rank's)."""
    import torch
    if dist is None:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
