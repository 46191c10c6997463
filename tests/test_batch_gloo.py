"""CPU, world_size 2 (gloo): the multi-GPU batch scheduler's sharding and result
gather (paper_1810_08218_b200/batch.py) with an injected solver standing in for
the GPU kernel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_08218_b200 import batch


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_solve(mesh, queries, out):
    # field of query [s] = s + 0.5 * vertex index (distinct per query and vertex)
    for i, q in enumerate(queries):
        out[i] = float(q[0]) + 0.5 * torch.arange(out.shape[1], dtype=out.dtype)
    return [{"source": q[0]} for q in queries]


def worker(rank, world, port, nq, n, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    queries = [[3 * q + 1] for q in range(nq)]
    fields, stats = batch.run_sharded(None, queries, n_vertices=n, device=torch.device("cpu"),
                                      solve=fake_solve)
    assert [s["source"] for s in stats] == [queries[q][0] for q in batch.shard(nq, world, rank)]
    if rank == 0:
        ret.put(fields.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("nq", [7, 8, 1])
def test_sharded_gather_world2(nq):
    world, n = 2, 11
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, nq, n, ret)) for r in range(world)]
    for p in procs:
        p.start()
    got = ret.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.stack([3 * q + 1 + 0.5 * np.arange(n) for q in range(nq)])
    assert np.array_equal(got, want.astype(np.float32))


def test_shard_partition():
    for nq in (0, 1, 5, 512):
        for world in (1, 2, 4, 8):
            parts = [batch.shard(nq, world, r) for r in range(world)]
            assert sorted(sum(parts, [])) == list(range(nq))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    assert batch.even_sources(1000, 4) == [[0], [250], [500], [750]]


def gpu_worker(rank, world, port, ret):
    """One rank of the real sharded batch: the B200 solver on cuda:0 (both ranks share
    the device), gloo for the gather (the BENCH_FORCE_DEVICE / BENCH_DIST_BACKEND=gloo
    configuration of bench.py)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_1810_08218_b200 as g
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v, f = g.noisy_icosphere_arrays(5, 2e-3, 1)
    M = g.Mesh(v, f, device=0)
    queries = batch.even_sources(len(v), 7)
    fields, stats = batch.run_sharded(M, queries, precision="single", groups=2)
    assert len(stats) == len(batch.shard(len(queries), world, rank))
    if rank == 0:
        ret.put(fields.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_real_solver_world2():
    """world_size 2 over gloo with the real GPU solve on one device: the gathered fields
    equal single-query runs bit for bit."""
    import paper_1810_08218_b200 as g
    world = 2
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=gpu_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    got = ret.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    v, f = g.noisy_icosphere_arrays(5, 2e-3, 1)
    M = g.Mesh(v, f)
    for q, src in enumerate(batch.even_sources(len(v), 7)):
        one = g.geodesics(M, src, precision="single")
        assert np.array_equal(got[q].astype(np.float64).view(np.int64),
                              one["distances"].view(np.int64)), q
