"""Multi-GPU partition logic, exercised on CPU with the gloo backend
(world_size 2): ranks own z-slabs, compute independently (the CPU oracle
stands in for the CUDA kernel here), and the concatenation equals the
single-process result; timing is reduced with a MAX over ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_07042_b200.sharding import World, slab_elements, slab_layers


@pytest.mark.parametrize("ez,ws", [(96, 1), (96, 2), (96, 4), (96, 8), (7, 3), (10, 4), (5, 5)])
def test_slabs_partition_the_layers(ez, ws):
    ranges = [slab_layers(ez, ws, r) for r in range(ws)]
    assert ranges[0][0] == 0 and ranges[-1][1] == ez
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a1 > a0
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_slab_elements_are_contiguous():
    counts = (4, 3, 6)
    got = [slab_elements(counts, 3, r) for r in range(3)]
    assert got == [(0, 24), (24, 48), (48, 72)]


def test_bad_world():
    with pytest.raises(ValueError):
        slab_layers(3, 4, 0)
    with pytest.raises(ValueError):
        slab_layers(8, 2, 2)


def test_world_from_env():
    w = World({"WORLD_SIZE": "4", "RANK": "2", "LOCAL_RANK": "1"})
    assert (w.size, w.rank, w.local_rank) == (4, 2, 1)
    assert World({}).max(3.5) == 3.5  # single process: identity


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    from oracle import hosfem_oracle as O
    from paper_2504_07042_b200.mesh import box_mesh

    world = World().init("gloo")
    order = 3
    mesh = box_mesh(3, 2, 4, order, perturbation=0.15, seed=2)
    e0, e1 = slab_elements(mesh.counts, ws, rank)
    z0, z1 = slab_layers(mesh.counts[2], ws, rank)
    verts = mesh.vertices_slab(z0, z1)
    assert verts.shape[0] == e1 - e0
    rng = np.random.default_rng(5)
    x_full = rng.standard_normal((mesh.n_elements, (order + 1) ** 3, 1))
    y = O.apply("trilinear", "poisson", order, verts, x_full[e0:e1])
    parts = [None] * ws
    dist.all_gather_object(parts, (e0, y))
    slowest = world.max(float(rank + 1))
    world.barrier()
    if rank == 0:
        parts.sort(key=lambda p: p[0])
        y_sharded = np.concatenate([p[1] for p in parts])
        y_full = O.apply("trilinear", "poisson", order, mesh.vertices, x_full)
        out.put((bool(np.array_equal(y_sharded, y_full)), slowest))
    world.close()


def test_two_rank_gloo_sharded_apply_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    equal, slowest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert equal
    assert slowest == 2.0
