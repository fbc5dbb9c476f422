"""Multi-rank parity on ONE GPU (P14, decomposition invariance; rows a6, a7):
P = 2, 3, 4 x-slab contexts of one process share the device through the
loopback transport (pic_loopback_link).  Each context runs on its own stream,
driven by its own host thread like a rank, and the peer transport's kernels
run unchanged: the mover writes slab leavers into the neighbour's receive
buffer (send_leavers_peer), event-handshake barriers publish them, arrive_kernel
appends and ranks them, ghost_pull_kernel sums the shared node planes, and
pic_implicit_sources reads the neighbour's planes.  The union of the slabs is
compared with the single-process CPU oracle (exiting
particles are transferred, a second kernel interpolates the received ones).
"""
import functools
import threading

import numpy as np
import pytest
import torch

import slab_parity as SP
from paper_2507_20719_b200 import decomp, inputs as I, pic

pytestmark = pytest.mark.gpu

CASES = {
    "c1r": (lambda: I.c1(randomized=True), 4, None),
    "c2s": (lambda: I.c2(nx_per_rank=32, ppc=27), 3, None),
    "c4inj": (lambda: I.c4(ncell=(32, 16, 16), ppc=8), 3, {"ppc": 8, "drift": (0.15, 0.0, 0.0)}),
    "c5s": (lambda: I.c5(ncell=(64, 32, 32), wind_ppc=2, inner_ppc=1, planet_ppc=16), 3, None),
}


@functools.lru_cache(maxsize=None)
def _oracle(name):
    make, cycles, inject = CASES[name]
    w = make()
    parts_all = I.make_species(w.with_slab(0, w.ncell[0]), device="cpu")
    return SP.oracle_reference(w, parts_all, cycles, inject)


def run_loopback(w, cycles, world, kernel, inject=None, bounds=None, sources=True, far_hops=0, check=True):
    """The loopback decomposition of workload w: returns gathered[r] =
    ([(particles, moments)] per species, stats, sources) like mr_parity."""
    bounds = bounds or decomp.uniform_bounds(w.ncell[0], world)
    parts_all, per_rank = SP.split_inputs(w, bounds)
    cap = SP.capacity(parts_all)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ctxs = []
    for r in range(world):
        wr = w.with_slab(bounds[r], bounds[r + 1])
        cfg = pic.make_config(wr, rank=r, nranks=world, capacity=cap, ghost=2, kernel=kernel,
                              transport=pic.TRANSPORT_LOOPBACK, far_hops=far_hops)
        ctx = pic.Context(cfg, stream=streams[r])
        dev = [{k: v.cuda() for k, v in p.items()} for p in per_rank[r]]
        _, EB = I.field_window(wr, 2, device="cpu")
        EB = EB.cuda()
        torch.cuda.synchronize()      # torch's copies before libpic's stream reads them
        for s, p in enumerate(dev):
            ctx.set_particles(s, p)
            if inject:
                ctx.set_injection(s, inject["ppc"], w.species[s].vth, inject["drift"], float(parts_all[s]["q"][0]),
                                  500 + s)
        ctx.set_fields(EB)
        ctxs.append(ctx)
    pic.pic_loopback_link(ctxs)
    assert all(c.transport == pic.TRANSPORT_LOOPBACK for c in ctxs)
    torch.cuda.synchronize()
    out = [None] * world
    errs = []

    def rank_body(r):
        try:
            with torch.cuda.stream(streams[r]):
                ctx = ctxs[r]
                for _ in range(cycles):
                    ctx.cycle()
                stats = ctx.sync(raise_on_error=check)
                src = tuple(t.cpu().numpy() for t in ctx.implicit_sources()) if sources else None
                out[r] = (stats, src)
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=rank_body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a loopback rank hung"
    assert not errs, errs
    torch.cuda.synchronize()
    gathered = []
    for r in range(world):
        local = []
        for s in range(len(w.species)):
            gp = {k: v.cpu().numpy() for k, v in ctxs[r].get_particles(s).items()}
            gm = ctxs[r].get_moments(s).cpu().numpy()
            local.append((gp, gm))
        gathered.append((local, out[r][0], out[r][1]))
    for c in ctxs:
        c.close()
    return gathered, parts_all


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("kernel", [pic.KERNEL_TILED, pic.KERNEL_BASIC])
@pytest.mark.parametrize("name", ["c1r", "c2s", "c4inj"])
def test_loopback_parity(name, kernel, world):
    make, cycles, inject = CASES[name]
    w = make()
    gathered, _ = run_loopback(w, cycles, world, kernel, inject=inject)
    ok, reps = SP.check_union(name, w, gathered, _oracle(name), kernel=kernel, transport="loopback", world=world)
    assert ok, reps
    # the exchange really ran: particles crossed slab faces both ways and arrived
    sent = sum(g[1]["sent"] for g in gathered)
    recv = sum(g[1]["received"] for g in gathered)
    assert sent > 0 and sent == recv, (sent, recv)
    assert any("sources_ok" in r for r in reps)


def test_loopback_parity_balanced_c5():
    """C5 clone (4 species, non-uniform ppc) on count-balanced slabs (H10)."""
    make, cycles, inject = CASES["c5s"]
    w = make()
    pc = I.plane_counts(w)
    bounds = decomp.balanced_bounds(pc.tolist(), 3, min_width=3)
    assert bounds != decomp.uniform_bounds(w.ncell[0], 3)
    gathered, _ = run_loopback(w, cycles, 3, pic.KERNEL_TILED, bounds=bounds)
    ok, reps = SP.check_union("c5s", w, gathered, _oracle("c5s"), kernel=pic.KERNEL_TILED, transport="loopback",
                              world=3)
    assert ok, reps


def test_loopback_ghost_planes_carry_the_stencil_overlap():
    """A particle just left of a slab face deposits into the right neighbour's
    first owned node plane; only the ghost-plane sum puts it there (a6)."""
    w = I.c1(randomized=True)
    gathered, parts_all = run_loopback(w, 1, 2, pic.KERNEL_TILED, sources=False)
    orc = _oracle_cycles(w, parts_all, 1)
    ok, reps = SP.check_union("c1r-1", w, gathered, orc, kernel=pic.KERNEL_TILED, transport="loopback", world=2)
    assert ok, reps
    # the owned plane x = slab_lo of rank 1 holds charge from both sides
    rho1 = gathered[1][0][0][1][0][:, :, 0]
    assert np.count_nonzero(rho1) > 0


def _oracle_cycles(w, parts_all, cycles):
    return SP.oracle_reference(w, parts_all, cycles)


def test_loopback_link_rejects_bad_groups():
    w = I.c1()
    bounds = decomp.uniform_bounds(w.ncell[0], 2)
    cfgs = [pic.make_config(w.with_slab(bounds[r], bounds[r + 1]), rank=r, nranks=2, capacity=[1024, 1024],
                            transport=pic.TRANSPORT_LOOPBACK) for r in range(2)]
    s = torch.cuda.Stream()
    a = pic.Context(cfgs[0], stream=s)
    b = pic.Context(cfgs[1], stream=s)
    with pytest.raises(pic.PicError):
        pic.pic_loopback_link([b, a])        # wrong rank order
    pic.pic_loopback_link([a, b])
    with pytest.raises(pic.PicError):
        pic.pic_loopback_link([a, b])        # twice
    _, EB = I.field_window(w.with_slab(bounds[0], bounds[1]), 2, device="cuda")
    a.set_fields(EB)
    with pytest.raises(pic.PicError) as e:
        a.mover(-1)                          # shared stream: the barriers would deadlock
    assert e.value.status == pic.PIC_EINVAL
    a.close()
    b.close()


def _with_fast_particles(w, n_fast=24, seed=9):
    """The workload's particles plus particles that cross 1.5 to 2.5 slabs of a
    P = 4 split in one step (6 to 10 cells along +-x)."""
    base = I.make_species
    def make(wl, device="cpu"):
        parts = base(wl, device=device)
        g = torch.Generator().manual_seed(seed)
        out = []
        for s, p in enumerate(parts):
            n = n_fast
            cells = 6 + 4 * torch.rand(n, generator=g, dtype=torch.float64)
            sign = torch.where(torch.rand(n, generator=g) < 0.5, -1.0, 1.0).to(torch.float64)
            u = sign * cells * w.delta[0] / w.dt
            extra = {"x": torch.rand(n, generator=g, dtype=torch.float64) * w.length[0],
                     "y": torch.rand(n, generator=g, dtype=torch.float64) * w.length[1],
                     "z": torch.rand(n, generator=g, dtype=torch.float64) * w.length[2],
                     "u": u, "v": torch.zeros(n, dtype=torch.float64), "w": torch.zeros(n, dtype=torch.float64),
                     "q": p["q"][:n].clone(), "id": torch.arange(n, dtype=torch.int64) + (1 << 52) + 1000 * s}
            out.append({k: torch.cat([p[k], extra[k].to(p[k].device)]).contiguous() for k in p})
        return out
    return make


@pytest.mark.parametrize("kernel", [pic.KERNEL_TILED, pic.KERNEL_BASIC])
def test_loopback_far_flyers_are_forwarded(kernel):
    """R22: particles that cross more than one slab in one step reach their
    owner through far_hops forwarding rounds (each receiver passes a record it
    does not own onward in its direction of motion) and match the oracle.
    Uniform fields (C1), so an iterate sampled beyond the field window (clamped,
    R11) sees the same field as the oracle's."""
    w = I.c1()
    orig = I.make_species
    I.make_species = _with_fast_particles(w)
    try:
        gathered, parts_all = run_loopback(w, 2, 4, kernel, sources=False, far_hops=2)
    finally:
        I.make_species = orig
    orc = SP.oracle_reference(w, parts_all, 2)
    ok, reps = SP.check_union("c1-far", w, gathered, orc, kernel=kernel, transport="loopback", world=4)
    assert ok, reps
    assert sum(g[1]["far"] for g in gathered) == 0
    assert sum(g[1]["sent"] for g in gathered) == sum(g[1]["received"] for g in gathered)


def test_loopback_far_flyers_without_forwarding_are_reported():
    w = I.c1()
    orig = I.make_species
    I.make_species = _with_fast_particles(w)
    try:
        gathered, _ = run_loopback(w, 1, 4, pic.KERNEL_TILED, sources=False, far_hops=0, check=False)
    finally:
        I.make_species = orig
    assert sum(g[1]["far"] for g in gathered) > 0


def test_loopback_barrier_timeout_is_an_error_not_a_hang():
    """A neighbour that never reaches the barrier: pic_mover reports PIC_ENCCL
    after barrier_timeout_ms instead of waiting forever."""
    import time
    w = I.c1()
    bounds = decomp.uniform_bounds(w.ncell[0], 2)
    parts_all, per_rank = SP.split_inputs(w, bounds)
    ctxs = []
    for r in range(2):
        wr = w.with_slab(bounds[r], bounds[r + 1])
        cfg = pic.make_config(wr, rank=r, nranks=2, capacity=SP.capacity(parts_all), transport=pic.TRANSPORT_LOOPBACK,
                              barrier_timeout_ms=500)
        ctx = pic.Context(cfg, stream=torch.cuda.Stream())
        dev = [{k: v.cuda() for k, v in p.items()} for p in per_rank[r]]
        EB = I.field_window(wr, 2, device="cuda")[1]
        torch.cuda.synchronize()
        for s, p in enumerate(dev):
            ctx.set_particles(s, p)
        ctx.set_fields(EB)
        ctxs.append(ctx)
    pic.pic_loopback_link(ctxs)
    t0 = time.time()
    with pytest.raises(pic.PicError) as e:
        ctxs[0].mover(-1)            # rank 1 never moves
    assert e.value.status == pic.PIC_ENCCL
    assert 0.4 < time.time() - t0 < 10
    for c in ctxs:
        c.close()
