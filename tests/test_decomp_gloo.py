"""Slab decomposition host logic on CPU (no GPU): bounds, ownership, NCCL-id
broadcast over a gloo process group, and a world-size-2 (and 3) model of the
exchange protocol libpic ships (DESIGN.md §3 R15, §8):

  1. mover      every rank moves its own particles (oracle Eq. 2);
  2. migration  a particle whose new cell belongs to another slab is sent to
                that rank, which must be a slab NEIGHBOUR (R22: no far-flyers):
                point-to-point, count first, then the records; the receiver
                appends them (send_leavers_peer / arrive_kernel, or the NCCL
                transport's migrate);
  3. deposit    every rank deposits the particles it now owns (oracle Eq. 3),
                so each particle is deposited once, by its new owner;
  4. ghost sum  the only nodes two slabs share are the face planes: rank r's
                deposit into node plane x = slab_hi (its edge cells' stencil
                overlap) is sent to the right neighbour and added into that
                rank's owned plane x = slab_lo (ghost_pull_kernel).

The owned planes of the union must equal the single-process oracle's moments
within R19 and the particle multiset must be identical by id.
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


def _neighbours(rank, world, periodic):
    left = rank - 1 if rank > 0 else (world - 1 if periodic else -1)
    right = rank + 1 if rank < world - 1 else (0 if periodic else -1)
    return left, right


def _send_recv(arr_to, peer_to, peer_from, like):
    """Point-to-point exchange of one numpy array (count first, then payload)."""
    reqs = []
    if peer_to >= 0:
        n = torch.tensor([arr_to.shape[0]], dtype=torch.int64)
        reqs.append(dist.isend(n, peer_to))
    got = None
    if peer_from >= 0:
        n = torch.zeros(1, dtype=torch.int64)
        dist.recv(n, peer_from)
        got = np.zeros((int(n.item()),) + like.shape[1:], dtype=like.dtype)
    for r in reqs:
        r.wait()
    reqs = []
    if peer_to >= 0 and arr_to.shape[0]:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr_to)), peer_to))
    if peer_from >= 0 and got.shape[0]:
        t = torch.from_numpy(got)
        dist.recv(t, peer_from)
        got = t.numpy()
    for r in reqs:
        r.wait()
    return got


KEYS = ("x", "y", "z", "u", "v", "w", "q")


def _worker(rank, world, port, q, cycles):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = decomp.broadcast_nccl_id(lambda: b"x" * 128)
        assert nid == b"x" * 128
        w = I.c1(randomized=True)
        bounds = decomp.uniform_bounds(w.ncell[0], world)
        lo, hi = bounds[rank], bounds[rank + 1]
        left, right = _neighbours(rank, world, w.bc[0] == I.PERIODIC)
        g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c)
        flo, EB = I.field_window(w, 2)
        F = O.FieldWindow(flo, EB.numpy())
        parts_all = I.make_species(w)
        results = []
        for s, sp in enumerate(w.species):
            P = {k: v.numpy().copy() for k, v in parts_all[s].items()}
            cell = np.floor(P["x"] / w.delta[0]).astype(np.int64)
            own = decomp.owner_of_cells(torch.from_numpy(cell), bounds).numpy() == rank
            P = {k: v[own].copy() for k, v in P.items()}
            sent = 0
            for cyc in range(cycles):
                # 1. mover (every rank its own particles)
                st, bad = O.mover(g, F, sp.qom, w.n_iter, P)
                assert bad == 0 and np.all(st == O.ALIVE)
                # 2. migration to the new owner, which must be a neighbour
                cell = np.floor(P["x"] / w.delta[0]).astype(np.int64)
                owner = decomp.owner_of_cells(torch.from_numpy(cell), bounds).numpy()
                assert set(np.unique(owner).tolist()) <= {rank, left, right}, "far-flyer (R22)"
                rec = np.stack([P[k] for k in KEYS] + [P["id"].view(np.float64)], 1)
                stay = owner == rank
                toL = rec[(owner == left) & ~stay] if left >= 0 else rec[:0]
                toR = rec[(owner == right) & ~stay & (owner != left)] if right >= 0 else rec[:0]
                sent += len(toL) + len(toR)
                # per-peer order: to the right / from the left, then to the left / from the right
                fromL = _send_recv(toR, right, left, rec)
                fromR = _send_recv(toL, left, right, rec)
                parts = [rec[stay]] + [a for a in (fromL, fromR) if a is not None]
                rec = np.concatenate(parts, 0)
                P = {k: rec[:, i].copy() for i, k in enumerate(KEYS)}
                P["id"] = rec[:, 7].copy().view(np.int64)
            # 3. deposit of the particles this rank owns (global periodic node grid)
            mom, am = O.moments(g, P)
            # 4. ghost sum: my node plane x = hi goes to the right neighbour's plane x = lo
            Nx = w.ncell[0]
            mine = mom[..., lo:hi].copy()
            amine = am[..., lo:hi].copy()
            edge = np.ascontiguousarray(np.stack([mom[..., hi % Nx], am[..., hi % Nx]], 0))[None]
            got = _send_recv(edge, right, left, edge)
            if got is not None:
                mine[..., 0] += got[0, 0]
                amine[..., 0] += got[0, 1]
            results.append(({k: v for k, v in P.items()}, mine, amine, sent))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_is_decomposition_invariant(world):
    cycles = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, cycles)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle
    w = I.c1(randomized=True)
    g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c)
    flo, EB = I.field_window(w, 2)
    F = O.FieldWindow(flo, EB.numpy())
    parts_all = I.make_species(w)
    for s, sp in enumerate(w.species):
        P = {k: v.numpy().copy() for k, v in parts_all[s].items()}
        for _ in range(cycles):
            st, _ = O.mover(g, F, sp.qom, w.n_iter, P)
        mom, am = O.moments(g, P, st)
        assert sum(out[r][s][3] for r in range(world)) > 0, "no particle crossed a slab face"
        ids = np.concatenate([out[r][s][0]["id"] for r in range(world)])
        assert np.array_equal(np.sort(ids), np.sort(P["id"]))
        merged = {k: np.concatenate([out[r][s][0][k] for r in range(world)]) for k in P}
        o1, o2 = np.argsort(merged["id"]), np.argsort(P["id"])
        for k in "xyzuvw":
            assert np.array_equal(merged[k][o1], P[k][o2])
        union = np.concatenate([out[r][s][1] for r in range(world)], axis=-1)
        assert union.shape == mom.shape
        assert np.all(np.abs(union - mom) <= 1e-10 * am)
        assert np.all(union[am == 0] == 0)


def test_ghost_sum_is_needed():
    """Without step 4 the owned face planes miss their left neighbour's edge
    cells' share: the protocol model is not trivially satisfied."""
    w = I.c1(randomized=True)
    g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c)
    parts = {k: v.numpy().copy() for k, v in I.make_species(w)[0].items()}
    cell = np.floor(parts["x"] / w.delta[0]).astype(np.int64)
    left = {k: v[cell < 8] for k, v in parts.items()}
    mom_all, _ = O.moments(g, parts)
    mom_right_only, _ = O.moments(g, {k: v[cell >= 8] for k, v in parts.items()})
    mom_left_only, _ = O.moments(g, left)
    assert np.any(mom_left_only[..., 8] != 0)            # left slab reaches plane 8
    assert not np.allclose(mom_right_only[..., 8], mom_all[..., 8])
