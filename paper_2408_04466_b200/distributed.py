"""Multi-GPU sharding: queries split across ranks, scene replicated, one
all-gather of the packed (w, status) block.  SURVEY.md §8(e): queries are independent, so the
data path has exactly one collective -- NCCL all-gather over NVLink on B200
boxes, gloo in the CPU tests.

Every rank builds the same scene deterministically (6.3 MB of control nets at
config 5) and evaluates the contiguous slice
``[rank*per, min(n, (rank+1)*per))``, ``per = ceil(n / world)``, passing the
slice's global start as ``index_base`` so jitter sequences -- and therefore
results -- are bit-identical to a single-GPU run.
"""

from __future__ import annotations

import math

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int, int]:
    per = max(1, math.ceil(n / world)) if n else 0
    s = min(n, rank * per)
    e = min(n, s + per)
    return s, e, per


def packed_shard(per: int, device):
    """This rank's send buffer for the one all-gather: ``per`` float64 winding
    numbers followed by ``per`` int8 status codes in one byte buffer
    (``per`` rounded up to a multiple of 8 so every rank's float64 block stays
    8-byte aligned in the gathered buffer).  Returns ``(buf, w_view, st_view)``;
    the engine writes straight into the views (no staging copy)."""
    import torch

    per8 = (per + 7) // 8 * 8
    buf = torch.zeros(9 * per8, dtype=torch.uint8, device=device)
    w_view = buf[: 8 * per8].view(torch.float64)
    st_view = buf[8 * per8:].view(torch.int8)
    st_view.fill_(-1)  # padding slots past the rank's slice
    return buf, w_view, st_view


def gather_packed(buf, world: int, n: int, *, group=None, out=None):
    """ONE all-gather of every rank's packed (w, status) block;
    returns full-length ``(w, status)`` in global query order.  ``out`` may
    pass a preallocated (world * len(buf),) uint8 receive buffer."""
    import torch
    import torch.distributed as dist

    if out is None:
        out = torch.empty(world * buf.numel(), dtype=torch.uint8, device=buf.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    per8 = buf.numel() // 9
    blocks = out.view(world, 9 * per8)
    w = blocks[:, : 8 * per8].reshape(-1).view(torch.float64).reshape(world, per8)
    st = blocks[:, 8 * per8:].view(torch.int8)
    return w, st


def unpad(w, st, per: int, n: int):
    """(world, per8) gathered blocks -> flat length-n results."""
    return w[:, :per].reshape(-1)[:n], st[:, :per].reshape(-1)[:n]


def sharded_winding_numbers(scene, queries, *, group=None, evaluate=None, device=None):
    """Evaluate this rank's slice of ``queries`` and all-gather the results.

    ``queries`` is the full (n,3) array on every rank (numpy or torch).
    ``evaluate(scene, local, index_base) -> (w, status)`` defaults to the
    B200 engine.  Returns full-length torch tensors ``(w, status)`` on
    ``device`` (the rank's CUDA device for NCCL, CPU for gloo).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = int(queries.shape[0])
    s, e, per = shard_bounds(n, rank, world)
    if evaluate is None:
        from .engine import winding_numbers

        def evaluate(sc, q, index_base):
            return winding_numbers(sc, q, index_base=index_base)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf, w_view, st_view = packed_shard(per, device)
    w_loc, st_loc = evaluate(scene, queries[s:e], s)
    w_view[: e - s] = torch.as_tensor(
        np.asarray(w_loc) if not torch.is_tensor(w_loc) else w_loc, dtype=torch.float64).to(device)
    st_view[: e - s] = torch.as_tensor(
        np.asarray(st_loc) if not torch.is_tensor(st_loc) else st_loc, dtype=torch.int8).to(device)
    w_all, st_all = gather_packed(buf, world, n, group=group)
    return unpad(w_all, st_all, per, n)
