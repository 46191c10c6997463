"""Batch scheduler for independent source queries across GPUs.

One process per GPU (torchrun), each holding a full mesh replica.  Queries are
dealt round-robin over the ranks (query q -> rank q % world, balancing the
source-dependent work), every rank solves its share with ONE persistent
launch (`geodist_batch_device`: several queries in flight per GPU as CTA
groups with separate barriers), and the per-query distance fields are
gathered to the destination rank over NCCL.  There is no collective inside a
solve: a single field never spans GPUs.

The gather is the only data-path collective.  `solve` is injectable so the
sharding and gather logic can be exercised with the gloo backend on CPU.
"""

import numpy as np


def shard(nq, world, rank):
    """Query indices of `rank` (round-robin)."""
    return list(range(rank, nq, world))


def local_count(nq, world, rank):
    return len(range(rank, nq, world))


def _device_solve(mesh, queries, out, precision, groups, epsilon):
    from . import batch_geodesics_device
    if len(queries) == 0:
        return []
    return batch_geodesics_device(mesh, queries, out.data_ptr(), epsilon=epsilon,
                                  precision=precision, groups=groups)


def run_sharded(mesh, queries, precision="single", groups=0, epsilon=1e-3, dst=0,
                n_vertices=None, device=None, solve=None, dist=None):
    """Solve `queries` (list of source lists) over all ranks of the default process
    group; returns (fields, stats) on `dst` -- fields is a [nq, n] tensor in query
    order on the destination's device -- and (None, local_stats) elsewhere.

    solve(mesh, local_queries, out_tensor) -> list of per-query stats fills
    out_tensor[i] with the field of local_queries[i] (default: the B200 kernel)."""
    import torch
    if dist is None:
        import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    n = n_vertices if n_vertices is not None else mesh.n_vertices
    dtype = torch.float32 if precision == "single" else torch.float64
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    nq = len(queries)
    mine = shard(nq, world, rank)
    per = (nq + world - 1) // world  # padded rows per rank for the collective
    local = torch.empty((max(per, 1), n), dtype=dtype, device=dev)
    if solve is None:
        stats = _device_solve(mesh, [queries[q] for q in mine], local, precision, groups, epsilon)
    else:
        stats = solve(mesh, [queries[q] for q in mine], local)
    if world == 1:
        return local[:nq], stats
    # NCCL gathers device buffers over NVLink; gloo (CPU tests) needs host copies
    send = local if dist.get_backend() == "nccl" else local.cpu()
    gathered = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, gathered, dst=dst)
    if rank != dst:
        return None, stats
    out = torch.empty((nq, n), dtype=dtype, device=dev)
    for r in range(world):
        idx = shard(nq, world, r)
        if idx:
            out[torch.as_tensor(idx, device=dev)] = gathered[r][:len(idx)].to(dev)
    return out, stats


def even_sources(n, count):
    """s_q = q * floor(n / count)."""
    step = max(1, n // count)
    return [[int(q * step)] for q in range(count)]


def as_numpy(fields):
    return None if fields is None else fields.detach().cpu().numpy().astype(np.float64)
