"""BP5 / Nekbone host logic on CPU: the oracle against the reference's own
Nekbone results, and the solver driver (slab layout, interface exchange,
rank-ordered reductions, CG) with a numpy backend, single rank and 2 ranks
under gloo."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import hosfem_oracle as O


def _nek(golden):
    return json.loads(bytes(golden["nekbone_json"]).decode())


def test_oracle_nekbone_matches_reference_golden(golden):
    for cfg in _nek(golden):
        got = O.nekbone(cfg["order"], tuple(cfg["elements"]), cfg["equation"], cfg["n_col"], cfg["perturbation"],
                        tol=1e-8, max_iter=300)
        for (src, it, err), want in zip(got, cfg["results"]):
            assert src == want["variant"] and it == want["iterations"]
            assert err == pytest.approx(want["error"], rel=1e-6)


def test_slab_layout_partitions_lattice():
    from paper_2504_07042_b200.solver import SlabLayout

    counts, order = (3, 2, 5), 2
    full = SlabLayout(counts, order)
    owned = 0
    for r in range(3):
        L = SlabLayout(counts, order, r, 3)
        s = L.global_slice()
        assert s.stop - s.start == L.n_local
        owned += L.n_owned
    assert owned == full.n_local == full.global_node_count


def _driver(order, elements, eq, n_col, pert, world=None):
    from paper_2504_07042_b200 import solver as S
    from bp5_numpy_backend import NumpyBackend

    cfg = S.NekboneConfig(order=order, elements=elements, equation=eq, n_col=n_col, perturbation=pert,
                          tol=1e-8, max_iter=300)
    res, _ = S.nekbone_benchmark(cfg, world=world, device="cpu", backend=NumpyBackend())
    return [(r.variant, r.iterations, r.error) for r in res]


def test_driver_single_rank_matches_reference(golden):
    """Our CG driver + numpy kernels reproduces the reference Nekbone runs."""
    for cfg in _nek(golden)[:3]:
        got = _driver(cfg["order"], tuple(cfg["elements"]), cfg["equation"], cfg["n_col"], cfg["perturbation"])
        for (src, it, err), want in zip(got, cfg["results"]):
            assert src == want["variant"]
            # the paper's Table 5 observable: same iteration count, same error level
            # (the final iterate's error moves at the 1% level under 1e-16 input changes)
            assert abs(it - want["iterations"]) <= 1
            assert err == pytest.approx(want["error"], rel=5e-2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    from paper_2504_07042_b200.sharding import World

    world = World().init("gloo")
    got = _driver(3, (3, 2, 4), "poisson", 1, 0.15, world=world)
    if rank == 0:
        q.put(got)
    world.close()


def test_two_rank_cg_matches_single_rank():
    """z-slab sharding with the interface exchange converges exactly like one rank."""
    single = _driver(3, (3, 2, 4), "poisson", 1, 0.15)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (s_src, s_it, s_err), (m_src, m_it, m_err) in zip(single, got):
        assert s_src == m_src and s_it == m_it
        assert m_err == pytest.approx(s_err, rel=1e-6)
