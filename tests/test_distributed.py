"""Multi-process host logic of the sharded path (gloo, world_size 2, CPU).

The device evaluation is stood in for by the CPU oracle (the checker), so
what is tested is the slicing, global index bases and the all-gather --
results must equal a single-process evaluation exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, n, out):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2408_04466_b200 import scenes
    from paper_2408_04466_b200.distributed import sharded_winding_numbers

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = scenes.make(cfg, n)

    def evaluate(sc, q, index_base):
        w, st, _, _ = O.scene_eval(s.ctrl, q, qidx=np.arange(index_base, index_base + len(q)),
                                   nthreads=2)
        return w, st

    w, st = sharded_winding_numbers(None, s.queries, evaluate=evaluate)
    if rank == 0:
        np.save(out + "_w.npy", w.numpy())
        np.save(out + "_st.npy", st.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n", [(1, 301), (2, 1000)])
def test_gloo_two_ranks_equal_single_process(tmp_path, cfg, n):
    from oracle import oracle as O
    from paper_2408_04466_b200 import scenes

    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), cfg, n, out), nprocs=2, join=True)
    w = np.load(out + "_w.npy")
    st = np.load(out + "_st.npy")
    s = scenes.make(cfg, n)
    w1, st1, _, _ = O.scene_eval(s.ctrl, s.queries, qidx=np.arange(n))
    assert w.shape == (n,)
    assert np.array_equal(w, w1) and np.array_equal(st, st1)


def test_shard_bounds_cover_exactly():
    from paper_2408_04466_b200.distributed import shard_bounds
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                s, e, per = shard_bounds(n, r, world)
                assert e - s <= per
                got.extend(range(s, e))
            assert got == list(range(n))


def _packed_worker(rank, world, port, n, out):
    import torch
    import torch.distributed as dist

    from paper_2408_04466_b200.distributed import gather_packed, packed_shard, shard_bounds, unpad

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e, per = shard_bounds(n, rank, world)
    buf, w_view, st_view = packed_shard(per, torch.device("cpu"))
    ids = torch.arange(s, e, dtype=torch.float64)
    w_view[: e - s] = ids * 0.5 - 3.25                 # any float64 bit pattern
    st_view[: e - s] = (torch.arange(s, e) % 4).to(torch.int8)  # status codes 0..3
    w, st = unpad(*gather_packed(buf, world, n), per, n)
    if rank == 0:
        np.save(out + "_w.npy", w.numpy())
        np.save(out + "_st.npy", st.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [13, 16, 1])
def test_packed_all_gather_one_collective(tmp_path, n):
    """(w, status) travel in ONE all-gather of a packed byte block per rank;
    ragged slices (per not a multiple of 8) and nonzero status codes."""
    out = str(tmp_path / "packed")
    mp.spawn(_packed_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
    w = np.load(out + "_w.npy")
    st = np.load(out + "_st.npy")
    ids = np.arange(n)
    assert w.dtype == np.float64 and st.dtype == np.int8
    assert np.array_equal(w, ids * 0.5 - 3.25)
    assert np.array_equal(st, (ids % 4).astype(np.int8))
