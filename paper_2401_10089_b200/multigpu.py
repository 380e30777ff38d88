"""Batch sharding across GPUs: matrices are independent units, so a batch
is split into contiguous chunks, one per rank/device, with no data-path collective.  The only
communication is the optional result gather at the end (reports and L to one rank).

Two modes:
* one process per GPU (torchrun, NCCL): ``shard_bounds`` + ``run_sharded`` -- each rank runs
  ``logm_batched`` on its chunk of its own device and ``gather_to`` collects (L, reports) on
  the destination rank with ``torch.distributed.gather_object`` (works over NCCL or gloo);
* one process driving several devices: ``driver.logm_batched(A, devices=[...])`` uses the
  same ``shard_bounds`` and runs each chunk on its device's current stream.
"""
import numpy as np


def shard_bounds(batch, world):
    """Contiguous [lo, hi) chunk per rank; sizes differ by at most one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return [((r * batch) // world, ((r + 1) * batch) // world) for r in range(world)]


def local_shard(A, rank, world):
    lo, hi = shard_bounds(A.shape[0], world)[rank]
    return A[lo:hi], lo


def gather_to(local_L, local_reports, rank, world, dst=0, group=None):
    """Gather per-rank (L chunk as numpy, report records) to `dst` in rank order.
    Returns (L, reports) on dst, (None, None) elsewhere."""
    import torch.distributed as dist

    payload = (np.asarray(local_L), np.asarray(local_reports))
    if world == 1:
        return payload
    objs = [None] * world if rank == dst else None
    dist.gather_object(payload, objs, dst=dst, group=group)
    if rank != dst:
        return None, None
    Ls = [o[0] for o in objs if o[0].shape[0]]
    Rs = [o[1] for o in objs if o[1].shape[0]]
    L = np.concatenate(Ls) if Ls else np.zeros((0,) + payload[0].shape[1:])
    R = np.concatenate(Rs) if Rs else payload[1][:0]
    return L, R


def run_sharded(A, rank, world, compute, dst=0, group=None):
    """Run ``compute(chunk) -> (L_chunk, reports_chunk)`` on this rank's contiguous chunk of
    the global batch ``A`` and gather the results to ``dst``."""
    chunk, _ = local_shard(A, rank, world)
    L, R = compute(chunk)
    return gather_to(L, R, rank, world, dst=dst, group=group)


def gather_tensor_to(local, rank, world, global_batch, dst=0, group=None):
    """Tensor gather of per-rank (b_r, ...) chunks to one (global_batch, ...) tensor on
    ``dst`` (rank order, contiguous shards as ``shard_bounds``).  Chunks are padded to the
    largest shard so one ``dist.gather`` moves them (NCCL over NVLink, or gloo); returns the
    gathered tensor on dst, None elsewhere.  world == 1 returns ``local`` unchanged."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    bounds = shard_bounds(global_batch, world)
    cap = max(hi - lo for lo, hi in bounds)
    lo, hi = bounds[rank]
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} items, shard is {hi - lo}")
    if local.shape[0] == cap:
        send = local.contiguous()
    else:
        send = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send[:local.shape[0]] = local
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([bufs[r][:hi_ - lo_] for r, (lo_, hi_) in enumerate(bounds)])
