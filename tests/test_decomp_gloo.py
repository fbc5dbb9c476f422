"""Slab decomposition host logic on CPU (no GPU): bounds, ownership, NCCL-id
broadcast over a gloo process group, and a world-size-2 model of the exchange
protocol (deposit-before-migrate into ghost planes, then migration) that must be
decomposition-invariant: identical particles by id and moments equal to the
single-process oracle within R19.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2507_20719_b200 import decomp
from paper_2507_20719_b200 import inputs as I


def test_uniform_bounds():
    assert decomp.uniform_bounds(16, 4) == [0, 4, 8, 12, 16]
    assert decomp.uniform_bounds(10, 3) == [0, 3, 6, 10]
    with pytest.raises(ValueError):
        decomp.uniform_bounds(2, 3)


def test_balanced_bounds():
    counts = [1.0] * 8 + [10.0] * 8
    b = decomp.balanced_bounds(counts, 2, min_width=2)
    assert b[0] == 0 and b[-1] == 16
    left = sum(counts[: b[1]])
    assert abs(left - sum(counts) / 2) <= 10
    b = decomp.balanced_bounds([0.0] * 4 + [5.0] * 12, 4, min_width=3)
    assert all(b[i + 1] - b[i] >= 3 for i in range(4))


def test_owner_of_cells_tie_goes_right():
    b = [0, 4, 8, 12]
    cx = torch.tensor([0, 3, 4, 7, 8, 11])
    assert decomp.owner_of_cells(cx, b).tolist() == [0, 0, 1, 1, 2, 2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = decomp.broadcast_nccl_id(lambda: b"x" * 128)
        assert nid == b"x" * 128
        w = I.c1(randomized=True)
        bounds = decomp.uniform_bounds(w.ncell[0], world)
        g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c)
        lo, EB = I.field_window(w, 2)
        F = O.FieldWindow(lo, EB.numpy())
        parts_all = I.make_species(w)
        results = []
        for s, sp in enumerate(w.species):
            P = {k: v.numpy().copy() for k, v in parts_all[s].items()}
            # this rank's slab at t = 0
            own = decomp.owner_of_cells(torch.from_numpy(np.floor(P["x"] / w.delta[0]).astype(np.int64)),
                                        bounds).numpy() == rank
            P = {k: v[own].copy() for k, v in P.items()}
            mom_tot = None
            for cyc in range(3):
                st, bad = O.mover(g, F, sp.qom, w.n_iter, P)
                assert bad == 0
                # deposit before migration (every rank deposits its own movers)
                mom, am = O.moments(g, P, st)
                # ghost sum == global reduction of the rank-local deposits
                t = torch.from_numpy(mom)
                dist.all_reduce(t)
                mom_tot = t.numpy()
                # migration by owner of the new cell
                cell = np.floor(P["x"] / w.delta[0]).astype(np.int64)
                owner = decomp.owner_of_cells(torch.from_numpy(cell), bounds).numpy()
                outgoing = [{k: v[owner == r] for k, v in P.items()} for r in range(world)]
                gathered = [None] * world
                dist.all_gather_object(gathered, outgoing)
                P = {k: np.concatenate([gathered[r][rank][k] for r in range(world)]) for k in P}
            results.append((P, mom_tot))
        q.put((rank, [({k: v for k, v in P.items()}, m) for P, m in results]))
    finally:
        dist.destroy_process_group()


def test_two_rank_protocol_is_decomposition_invariant():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle
    w = I.c1(randomized=True)
    g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c)
    lo, EB = I.field_window(w, 2)
    F = O.FieldWindow(lo, EB.numpy())
    parts_all = I.make_species(w)
    for s, sp in enumerate(w.species):
        P = {k: v.numpy().copy() for k, v in parts_all[s].items()}
        for _ in range(3):
            st, _ = O.mover(g, F, sp.qom, w.n_iter, P)
        mom, am = O.moments(g, P, st)
        ids = np.concatenate([out[r][s][0]["id"] for r in range(world)])
        assert np.array_equal(np.sort(ids), np.sort(P["id"]))
        merged = {k: np.concatenate([out[r][s][0][k] for r in range(world)]) for k in P}
        o1, o2 = np.argsort(merged["id"]), np.argsort(P["id"])
        for k in "xyzuvw":
            assert np.array_equal(merged[k][o1], P[k][o2])
        m2 = out[0][s][1]
        assert np.all(np.abs(m2 - mom) <= 1e-10 * am)
