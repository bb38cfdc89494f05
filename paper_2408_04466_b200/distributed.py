"""Multi-GPU sharding: queries split across ranks, scene replicated, one
all-gather of (w, status).  SURVEY.md §8(e): queries are independent, so the
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
    w_loc, st_loc = evaluate(scene, queries[s:e], s)
    w_loc = torch.as_tensor(np.asarray(w_loc) if not torch.is_tensor(w_loc) else w_loc,
                            dtype=torch.float64).to(device)
    st_loc = torch.as_tensor(np.asarray(st_loc) if not torch.is_tensor(st_loc) else st_loc,
                             dtype=torch.int8).to(device)
    w_pad = torch.zeros(per, dtype=torch.float64, device=device)
    st_pad = torch.full((per,), -1, dtype=torch.int8, device=device)
    w_pad[: e - s] = w_loc
    st_pad[: e - s] = st_loc
    w_all = torch.empty(per * world, dtype=torch.float64, device=device)
    st_all = torch.empty(per * world, dtype=torch.int8, device=device)
    dist.all_gather_into_tensor(w_all, w_pad, group=group)
    dist.all_gather_into_tensor(st_all, st_pad, group=group)
    return w_all[:n], st_all[:n]
