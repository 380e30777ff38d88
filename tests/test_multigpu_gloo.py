"""Multi-rank sharding/gather host logic on CPU: world_size 2 over gloo (127.0.0.1).

The GPU call is replaced by the CPU oracle as the per-rank compute (this exercises the
sharding, rank ordering and gather path, not the kernels); the gathered result must equal
the single-process run bit for bit, and every matrix must be covered exactly once.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_2401_10089_b200.multigpu import shard_bounds


def test_shard_bounds_cover_exactly():
    for batch in (0, 1, 7, 8, 4096, 4097):
        for world in (1, 2, 3, 8):
            b = shard_bounds(batch, world)
            assert b[0][0] == 0 and b[-1][1] == batch
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(chunk):
    from oracle import driver as D
    Ls, Rs = [], []
    for A in chunk:
        L, rep = D.logm_status(A, D.default_prims())
        Ls.append(L)
        Rs.append((rep["status"], rep["s"], rep["k"], rep["db_iters"], rep["estimation_passes"]))
    return np.stack(Ls), np.array(Rs, dtype=np.int64)


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2401_10089_b200 import synth
    from paper_2401_10089_b200.multigpu import run_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = synth.config(2, batch=9)
    L, R = run_sharded(A, rank, world, _oracle_compute)
    if rank == 0:
        np.savez(out_path, L=L, R=R)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather(tmp_path):
    from paper_2401_10089_b200 import synth
    out = str(tmp_path / "gathered.npz")
    port = _free_port()
    tmp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    A = synth.config(2, batch=9)
    L1, R1 = _oracle_compute(A)
    assert np.array_equal(got["L"], L1)
    assert np.array_equal(got["R"], R1)


def _tensor_worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    from paper_2401_10089_b200.multigpu import gather_tensor_to, shard_bounds as sb
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = 7                                             # unequal shards: 3 + 4
    full = torch.arange(G * 4, dtype=torch.float64).view(G, 2, 2)
    lo, hi = sb(G, world)[rank]
    got = gather_tensor_to(full[lo:hi].clone(), rank, world, G)
    if rank == 0:
        torch.save(got, out_path)
    else:
        assert got is None
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_tensor_gather_unequal_shards(tmp_path):
    import torch
    out = str(tmp_path / "t.pt")
    tmp.spawn(_tensor_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    assert torch.equal(got, torch.arange(28, dtype=torch.float64).view(7, 2, 2))
