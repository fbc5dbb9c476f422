"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Same seeded inputs on both sides (paper_2507_20719_b200.inputs), compared by
particle id with the north_star tolerances (tests/parity_util.py).  Sizes are
small enough for the oracle to finish in seconds while spanning many cells and
tiles, with ragged particle counts.
"""
import numpy as np
import pytest
import torch

from paper_2507_20719_b200 import inputs as I
from paper_2507_20719_b200 import pic
import parity_util as PU

pytestmark = pytest.mark.gpu


def run_gpu(w, parts, cycles, kernel, ghost=2, n_iter=None):
    cap = [int(p["x"].numel() * 1.25) + 64 for p in parts]
    cfg = pic.make_config(w, capacity=cap, ghost=ghost, kernel=kernel, n_iter=n_iter)
    ctx = pic.Context(cfg)
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    lo, EB = I.field_window(w, ghost, device="cpu")
    ctx.set_fields(EB.cuda())
    for _ in range(cycles):
        ctx.cycle()
    stats = ctx.sync()
    out = []
    for s in range(len(parts)):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        gm = ctx.get_moments(s).cpu().numpy()
        out.append((gp, gm))
    ctx.close()
    return out, stats


def check(w, cycles, kernel, ghost=2, n_iter=None):
    parts = I.make_species(w, device="cpu")
    orc = PU.run_oracle(w, parts, cycles, ghost=ghost, n_iter=n_iter)
    gpu, stats = run_gpu(w, parts, cycles, kernel, ghost, n_iter)
    reports = []
    import oracle as O
    g = PU.oracle_grid(w)
    for s, sp in enumerate(w.species):
        rep = {"species": sp.name}
        ok_p = PU.compare_particles(w, sp, gpu[s][0], orc[s][0], orc[s][1], rep)
        ok_m = PU.compare_moments(gpu[s][1], orc[s][2], orc[s][3], rep)
        # P13 two-level: the oracle's deposit of the GPU's own particles against
        # the GPU moments (isolates Eq. 3 from the mover)
        gp = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in gpu[s][0].items() if k != "id"}
        m2, a2 = O.moments(g, gp, None)
        rep2 = {}
        ok_d = PU.compare_moments(gpu[s][1], m2, a2, rep2)
        rep["deposit_only_ratio"] = rep2.get("mom_ratio")
        reports.append(rep)
        assert ok_p and ok_m and ok_d, rep
    return reports, stats


KERNELS = [pic.KERNEL_BASIC, pic.KERNEL_TILED]


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1_uniform(kernel):
    reps, stats = check(I.c1(), 5, kernel)
    assert stats["removed"] == 0 and stats["far"] == 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1r_random_fields(kernel):
    check(I.c1(randomized=True), 5, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c2_harris_scaled(kernel):
    # C2 structure at 1/8 size in x and reduced ppc (oracle in seconds)
    w = I.c2(nx_per_rank=16, ppc=27)
    check(w, 3, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c4_open_dipole_scaled(kernel):
    w = I.c4(ncell=(32, 16, 16), ppc=8)
    reps, stats = check(w, 4, kernel)
    assert stats["removed"] > 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1_relativistic(kernel):
    # NEXT-1: relativistic Eq. 2 (gamma up to ~2 for the electrons)
    w = I.c1rel()
    parts = I.make_species(w, device="cpu")
    g = 1.0 / torch.sqrt(1.0 - (parts[0]["u"] ** 2 + parts[0]["v"] ** 2 + parts[0]["w"] ** 2))
    assert float(g.max()) > 1.5
    check(w, 4, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c3_fourier_scaled(kernel):
    # C3 structure (B0 z + random Fourier modes, periodic cube) at 24^3, 8 ppc
    w = I.c3(n_per_rank=24, ppc=8)
    check(w, 3, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c5_four_species_nonuniform_ppc(kernel):
    # C5 structure at 1/8 size: 4 species, wind ppc 4/1 in/out of the
    # magnetosphere ellipsoid, planetary ppc round(32 exp(-(r-R)/2)), open BC
    w = I.c5(ncell=(64, 32, 32), wind_ppc=4, inner_ppc=1, planet_ppc=32)
    parts = I.make_species(w, device="cpu")
    assert len(parts) == 4 and parts[2]["x"].numel() > 0
    reps, stats = check(w, 3, kernel)
    assert stats["removed"] > 0


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("n_iter", [1, 2, 4, 5])
def test_n_iter_variants(n_iter, kernel):
    # 1, 2, 4: compile-time iteration counts of the tiled mover; 5: runtime count
    check(I.c1(randomized=True), 2, kernel, n_iter=n_iter)


def test_ragged_and_empty_species():
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    # ragged: drop a random subset of species 0, empty species 1
    g = torch.Generator().manual_seed(5)
    keep = torch.rand(parts[0]["x"].numel(), generator=g) < 0.37
    parts[0] = {k: v[keep].contiguous() for k, v in parts[0].items()}
    parts[1] = {k: v[:0].contiguous() for k, v in parts[1].items()}
    orc = PU.run_oracle(w, parts, 3)
    gpu, _ = run_gpu(w, parts, 3, pic.KERNEL_TILED)
    rep = {}
    assert PU.compare_particles(w, w.species[0], gpu[0][0], orc[0][0], orc[0][1], rep), rep
    assert PU.compare_moments(gpu[0][1], orc[0][2], orc[0][3], rep), rep
    assert gpu[1][0]["x"].size == 0 and not gpu[1][1].any()


def test_closed_form_gyration_on_gpu():
    """P2 on the GPU path directly: |v| conserved and the rotation angle per step."""
    import math
    w = I.c1()
    w.field_params = {"E": (0.0, 0.0, 0.0), "B": (0.0, 0.0, 0.01)}
    parts = I.make_species(w, device="cpu")
    gpu, _ = run_gpu(w, parts, 1, pic.KERNEL_TILED)
    for s, sp in enumerate(w.species):
        gp = gpu[s][0]
        order = np.argsort(gp["id"])
        p0 = {k: v.numpy() for k, v in parts[s].items()}
        o0 = np.argsort(p0["id"])
        v0 = np.stack([p0["u"][o0], p0["v"][o0]], 1)
        v1 = np.stack([gp["u"][order], gp["v"][order]], 1)
        th = 2 * math.atan(abs(sp.qom) * 0.01 * w.dt / 2)
        ang = np.arctan2(v0[:, 0] * v1[:, 1] - v0[:, 1] * v1[:, 0], (v0 * v1).sum(1))
        assert np.allclose(ang, -math.copysign(th, sp.qom), atol=1e-9)
        assert np.allclose(np.linalg.norm(v1, axis=1), np.linalg.norm(v0, axis=1), rtol=1e-13)


def test_call_order_errors():
    w = I.c1()
    parts = I.make_species(w, device="cpu")
    cfg = pic.make_config(w, capacity=[p["x"].numel() for p in parts])
    ctx = pic.Context(cfg)
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    with pytest.raises(pic.PicError) as e:
        ctx.mover()            # fields not set
    assert e.value.status == pic.PIC_ESTATE
    lo, EB = I.field_window(w, 2)
    ctx.set_fields(EB.cuda())
    with pytest.raises(pic.PicError) as e:
        ctx.exchange()         # before moments
    assert e.value.status == pic.PIC_ESTATE
    ctx.mover()
    with pytest.raises(pic.PicError) as e:
        ctx.mover()            # twice
    assert e.value.status == pic.PIC_ESTATE
    ctx.moments()
    ctx.exchange()
    ctx.sync()
    ctx.close()


def test_nonfinite_flag():
    w = I.c1()
    parts = I.make_species(w, device="cpu")
    cfg = pic.make_config(w, capacity=[p["x"].numel() for p in parts])
    ctx = pic.Context(cfg)
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    lo, EB = I.field_window(w, 2)
    EB[3, 3, 3, 0] = float("nan")
    ctx.set_fields(EB.cuda())
    ctx.cycle()
    with pytest.raises(pic.PicError) as e:
        ctx.sync()
    assert e.value.status == pic.PIC_ENONFINITE
    ctx.close()


def test_field_sequence_and_async_moments():
    """Fields change every cycle (double-buffered pic_set_fields from pinned host
    and device sources) and moments come back through pic_get_moments_async;
    the oracle runs the same field sequence."""
    import copy
    import oracle as O
    wa = I.c1(randomized=True)
    wb = copy.deepcopy(wa)
    wb.field_params["B"] = tuple(2.0 * b for b in wa.field_params["B"])
    wb.field_params["E"] = tuple(-3.0 * e for e in wa.field_params["E"])
    seq = [wa, wb, wa, wb]
    parts = I.make_species(wa, device="cpu")
    # oracle
    g = PU.oracle_grid(wa)
    Fs = {id(w): PU.oracle_field(w, 2) for w in (wa, wb)}
    orc = []
    for s, sp in enumerate(wa.species):
        P = PU.to_numpy_parts(parts[s])
        st = np.zeros(len(P["x"]), dtype=np.int8)
        for w in seq:
            st, bad = O.mover(g, Fs[id(w)], sp.qom, wa.n_iter, P, st)
            assert bad == 0
        mom, am = O.moments(g, P, st)
        orc.append((P, st, mom, am))
    # GPU
    cap = [int(p["x"].numel() * 1.25) + 64 for p in parts]
    ctx = pic.Context(pic.make_config(wa, capacity=cap, kernel=pic.KERNEL_TILED))
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    EB = {id(w): I.field_window(w, 2, device="cpu")[1] for w in (wa, wb)}
    EB_pinned = {k: v.pin_memory() for k, v in EB.items()}
    shape = ctx.moment_shape()
    outs = [torch.empty((10, shape[2], shape[1], shape[0]), dtype=torch.float64).pin_memory()
            for _ in wa.species]
    for i, w in enumerate(seq):
        ctx.set_fields(EB_pinned[id(w)] if i % 2 == 0 else EB[id(w)].cuda())
        ctx.cycle()
        for s in range(len(wa.species)):
            ctx.get_moments_async(s, outs[s])
    ctx.join_copies()
    ctx.sync()
    for s, sp in enumerate(wa.species):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        rep = {"species": sp.name}
        assert PU.compare_particles(wa, sp, gp, orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(outs[s].numpy(), orc[s][2], orc[s][3], rep), rep
        # the synchronous copy-out agrees bit for bit
        assert torch.equal(ctx.get_moments(s).cpu(), outs[s])
    ctx.close()


def _ctx_for(w, parts, kernel=pic.KERNEL_TILED, extra=64):
    ctx = pic.Context(pic.make_config(w, capacity=[p["x"].numel() + extra for p in parts], kernel=kernel))
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    ctx.set_fields(I.field_window(w, 2)[1].cuda())
    return ctx


@pytest.mark.parametrize("kernel", KERNELS)
def test_single_particle_and_sparse_tiles(kernel):
    """One particle per species in a 16^3 box (63 of 64 tiles empty): parity."""
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    parts = [{k: v[1234:1235].contiguous() for k, v in p.items()} for p in parts]
    orc = PU.run_oracle(w, parts, 3)
    gpu, _ = run_gpu(w, parts, 3, kernel)
    for s, sp in enumerate(w.species):
        rep = {}
        assert PU.compare_particles(w, sp, gpu[s][0], orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(gpu[s][1], orc[s][2], orc[s][3], rep), rep


@pytest.mark.parametrize("kernel", KERNELS)
def test_multiple_wrap_is_an_error(kernel):
    """R10: a particle that would wrap more than once in one step -> PIC_ERANGE."""
    w = I.c1()
    parts = I.make_species(w, device="cpu")
    parts[0]["u"][7] = 3.0 * w.length[0] / w.dt     # three box lengths per step
    ctx = _ctx_for(w, parts, kernel)
    ctx.cycle()
    with pytest.raises(pic.PicError) as e:
        ctx.sync()
    assert e.value.status == pic.PIC_ERANGE
    ctx.close()


def test_capacity_is_enforced():
    w = I.c1()
    parts = I.make_species(w, device="cpu")
    ctx = pic.Context(pic.make_config(w, capacity=[10, 10]))
    with pytest.raises(pic.PicError) as e:
        ctx.set_particles(0, {k: v.cuda() for k, v in parts[0].items()})
    assert e.value.status == pic.PIC_ERANGE
    ctx.close()


def test_open_boundary_removal_counts():
    """C4 clone: particles leaving through open faces or into the planet are
    removed; the live count plus the removed count is conserved."""
    w = I.c4(ncell=(32, 16, 16), ppc=8)
    parts = I.make_species(w, device="cpu")
    n0 = sum(p["x"].numel() for p in parts)
    ctx = _ctx_for(w, parts)
    for _ in range(6):
        ctx.cycle()
    stats = ctx.sync()
    n1 = sum(ctx.count(s) for s in range(len(parts)))
    assert stats["removed"] > 0 and n1 + stats["removed"] == n0
    ctx.close()


@pytest.mark.parametrize("cfg", ["c1r", "c4s"])
def test_implicit_sources_two_level(cfg):
    """NEXT-2 (Eq. 5-6): GPU chi, rho-hat, J-hat against the oracle fed with the
    GPU's own moments (two-level parity, P13: isolates the sources stencil; the
    moments themselves are pinned by the parity tests above)."""
    import oracle as O
    w = I.c1(randomized=True) if cfg == "c1r" else I.c4(ncell=(32, 16, 16), ppc=8)
    parts = I.make_species(w, device="cpu")
    ctx = _ctx_for(w, parts)
    for _ in range(2):
        ctx.cycle()
    ctx.sync()
    gm = [ctx.get_moments(s).cpu().numpy() for s in range(len(parts))]
    chi, rh, jh = (t.cpu().numpy() for t in ctx.implicit_sources())
    ctx.close()
    G = 2
    lo, EB = I.field_window(w, G)
    nz, ny, nx = gm[0].shape[1:]
    Bn = EB[G:G + nz, G:G + ny, G:G + nx, 3:6].numpy()
    g = PU.oracle_grid(w)
    ochi, orh, ojh = O.implicit_sources(g, [sp.qom for sp in w.species], gm, Bn)
    for got, want in ((chi, ochi), (rh, orh), (jh, ojh)):
        scale = np.abs(want).max()
        assert scale > 0
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("kernel", KERNELS)
def test_inflow_injection(kernel):
    """NEXT-3: inflow injection at the open x = 0 face (both species, drifting
    Maxwellian, Philox draws on both sides) over several cycles of a C4 clone;
    particles (incl. the injected ones, by id) and moments match the oracle."""
    import oracle as O
    w = I.c4(ncell=(32, 16, 16), ppc=8)
    parts = I.make_species(w, device="cpu")
    cycles, ppc, drift = 4, 8, (0.15, 0.01, -0.02)
    inj = [dict(ppc=ppc, vth=sp.vth, drift=drift, q=float(parts[s]["q"][0]), seed=1000 + 17 * s)
           for s, sp in enumerate(w.species)]
    g = PU.oracle_grid(w)
    F = PU.oracle_field(w, 2)
    orc = []
    for s, sp in enumerate(w.species):
        P = PU.to_numpy_parts(parts[s])
        st = np.zeros(len(P["x"]), dtype=np.int8)
        n_inj = 0
        for c in range(cycles):
            st, bad = O.mover(g, F, sp.qom, w.n_iter, P, st)
            assert bad == 0
            a = inj[s]
            new = O.inject(g, F, s, sp.qom, w.n_iter, a["seed"], c, a["ppc"], a["vth"], a["drift"], a["q"])
            n_inj += len(new["x"])
            P = {k: np.concatenate([P[k], new[k]]) for k in P}
            st = np.concatenate([st, np.zeros(len(new["x"]), dtype=np.int8)])
        assert n_inj > 100
        mom, am = O.moments(g, P, st)
        orc.append((P, st, mom, am))
    cap = [int(p["x"].numel() * 1.25) + cycles * 16 * 16 * ppc + 64 for p in parts]
    ctx = pic.Context(pic.make_config(w, capacity=cap, kernel=kernel))
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
        a = inj[s]
        ctx.set_injection(s, a["ppc"], a["vth"], a["drift"], a["q"], a["seed"])
    ctx.set_fields(I.field_window(w, 2)[1].cuda())
    for _ in range(cycles):
        ctx.cycle()
    ctx.sync()
    for s, sp in enumerate(w.species):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        gm = ctx.get_moments(s).cpu().numpy()
        rep = {"species": sp.name}
        assert PU.compare_particles(w, sp, gp, orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(gm, orc[s][2], orc[s][3], rep), rep
        assert (gp["id"] >> 62 == 1).sum() > 100
    ctx.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_particle_control(kernel):
    """NEXT-3 particle control between cycles: a split pass (target above the
    count) and a coalescence pass (target below), then more cycles; particles
    (children by their hashed ids, merged ones gone) and moments match the oracle
    running the same sequence."""
    import oracle as O
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    eps, seed = 0.1, 99
    dvs = [sp.vth / 2 for sp in w.species]
    # plan: (cycles, then control with target factor)
    plan = [(1, 1.3), (1, 0.8), (1, None)]
    g = PU.oracle_grid(w)
    F = PU.oracle_field(w, 2)
    orc = []
    for s, sp in enumerate(w.species):
        P = PU.to_numpy_parts(parts[s])
        st = np.zeros(len(P["x"]), dtype=np.int8)
        cyc = 0
        n0 = len(P["x"])
        for ncyc, fac in plan:
            for _ in range(ncyc):
                st, bad = O.mover(g, F, sp.qom, w.n_iter, P, st)
                assert bad == 0
                cyc += 1
            if fac is None:
                continue
            n = int((st == O.ALIVE).sum())
            target = int(fac * n0)
            if n < target * (1 - 0.05):
                P, st = O.split(g, s, P, st, min(1.0, (target - n) / n), eps, seed, cyc)
            elif n > target * (1 + 0.05):
                assert O.coalesce(g, P, st, dvs[s], (n - target) / n) > 0
        mom, am = O.moments(g, P, st)
        orc.append((P, st, mom, am))
    cap = [int(p["x"].numel() * 2.2) + 64 for p in parts]
    ctx = pic.Context(pic.make_config(w, capacity=cap, kernel=kernel))
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    ctx.set_fields(I.field_window(w, 2)[1].cuda())
    n0s = [p["x"].numel() for p in parts]
    acts = []
    for ncyc, fac in plan:
        for _ in range(ncyc):
            ctx.cycle()
        if fac is not None:
            acts.append([ctx.control(s, int(fac * n0s[s]), 0.05, eps, dvs[s], seed) for s in range(len(parts))])
    # the last cycle's moments are of the state after the last control pass + cycle
    ctx.sync()
    assert acts == [[1, 1], [2, 2]]
    for s, sp in enumerate(w.species):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        gm = ctx.get_moments(s).cpu().numpy()
        rep = {"species": sp.name}
        assert PU.compare_particles(w, sp, gp, orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(gm, orc[s][2], orc[s][3], rep), rep
    ctx.close()


@pytest.mark.parametrize("M", [1, 3])
def test_gmm_histogram_and_em(M):
    """NEXT-4: the GPU velocity histogram against the oracle's (same particles
    after two cycles) and the GPU EM fit against the oracle fed with the GPU's
    histogram (two-level)."""
    import oracle as O
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    orc = PU.run_oracle(w, parts, 2)
    ctx = _ctx_for(w, parts)
    for _ in range(2):
        ctx.cycle()
    ctx.sync()
    for s, sp in enumerate(w.species):
        B, vmax = 16, 4.0 * sp.vth
        a, mu, sg, h, clipped = ctx.gmm(s, B, vmax, M, 25)
        oh, oc = O.bin_velocities(orc[s][0], orc[s][1], B, vmax)
        assert clipped == oc
        np.testing.assert_allclose(h, oh, rtol=1e-12, atol=0)
        oa, omu, osg = O.fit_gmm(h, vmax, M, 25)
        np.testing.assert_allclose(a, oa, rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(mu, omu, rtol=1e-9, atol=1e-9 * vmax)
        np.testing.assert_allclose(sg, osg, rtol=1e-8, atol=1e-9 * vmax * vmax)
    ctx.close()


def test_moment_ptr_matches_copy_out():
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    ctx = _ctx_for(w, parts)
    ctx.cycle()
    ctx.sync()
    for s in range(len(parts)):
        full = ctx.get_moments(s)
        for comp in (0, 3, 9):
            raw, scale = ctx.moment_view(s, comp)
            assert raw.data_ptr() != full.data_ptr()
            assert torch.equal(raw * scale, full[comp])
    ctx.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_coalesce_overfull_and_wide_cells(kernel):
    """R31 on every cell ("in cells with an excessive number of
    particles, we perform pair-wise merging"): a 2000-particle cell and a cell
    whose velocity bins lie beyond +-2^20 (and +-3e12) take the unpacked
    global-memory path; the survivors match the oracle's coalescence exactly
    as the 27-particle cells do."""
    import oracle as O
    w = I.c1(randomized=True)
    base = I.make_species(w, device="cpu")[0]
    sp = w.species[0]
    dv = sp.vth / 2
    gen = torch.Generator().manual_seed(77)
    d = w.delta
    # 2000 extra particles in cell (5, 6, 7)
    n_big = 2000
    big = {"x": (5 + torch.rand(n_big, generator=gen, dtype=torch.float64)) * d[0],
           "y": (6 + torch.rand(n_big, generator=gen, dtype=torch.float64)) * d[1],
           "z": (7 + torch.rand(n_big, generator=gen, dtype=torch.float64)) * d[2]}
    for k in "uvw":
        big[k] = sp.vth * torch.randn(n_big, generator=gen, dtype=torch.float64)
    big["q"] = base["q"][:1].repeat(n_big) * (1 + 0.1 * torch.rand(n_big, generator=gen, dtype=torch.float64))
    big["id"] = 10**9 + torch.arange(n_big, dtype=torch.int64)
    # wide bins in cell (2, 3, 4): pairs at bin 2^21 and at 3e12, one at -2^21
    wide_u = torch.tensor([2**21 + 0.25, 2**21 + 0.5, 2**21 + 0.75, 3e12, 3e12 + 0.5, -2**21 - 0.5],
                          dtype=torch.float64) * dv
    nw = wide_u.numel()
    wide = {"x": torch.full((nw,), 2.5 * d[0], dtype=torch.float64) + 0.01 * torch.arange(nw) * d[0],
            "y": torch.full((nw,), 3.5 * d[1], dtype=torch.float64),
            "z": torch.full((nw,), 4.5 * d[2], dtype=torch.float64),
            "u": wide_u, "v": torch.full((nw,), 0.3 * dv, dtype=torch.float64),
            "w": torch.full((nw,), -0.3 * dv, dtype=torch.float64),
            "q": base["q"][:1].repeat(nw), "id": 2 * 10**9 + torch.arange(nw, dtype=torch.int64)}
    parts = {k: torch.cat([base[k], big[k], wide[k]]).contiguous() for k in base}
    n = parts["x"].numel()
    target = int(0.7 * n)
    frac = (n - target) / n
    # oracle: the same coalescence pass on the initial state
    g = PU.oracle_grid(w)
    P = PU.to_numpy_parts(parts)
    st = np.zeros(n, dtype=np.int8)
    merges = O.coalesce(g, P, st, dv, frac)
    assert merges > 0
    # the big cell and the wide cell both merged on the oracle side
    merged_ids = set(P["id"][st == O.MERGED].tolist())
    assert any(i >= 10**9 and i < 2 * 10**9 for i in merged_ids)
    assert {2 * 10**9 + 1, 2 * 10**9 + 4} <= merged_ids
    import dataclasses
    wq = pic.make_config(dataclasses.replace(w, species=[sp]), capacity=[n + 64], kernel=kernel)
    ctx = pic.Context(wq)
    ctx.set_particles(0, {k: v.cuda() for k, v in parts.items()})
    assert ctx.control(0, target, 0.05, 0.1, dv, 5) == 2
    ctx.sync()
    gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(0).items()}
    # the GPU keeps positions in cell units; compare by id
    assert len(gp["id"]) == int((st == O.ALIVE).sum())
    rep = {}
    assert PU.compare_particles(w, sp, gp, P, st, rep), rep
    ctx.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_graph_cycles_match_the_oracle(kernel):
    """pic_set_graph: cycles replayed from CUDA graphs (one per field buffer x
    store buffer parity; new fields every other cycle switch the field buffer)
    give the oracle's particles and moments like plain launches."""
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    cycles = 6
    orc = PU.run_oracle(w, parts, cycles)
    cap = [p["x"].numel() + 64 for p in parts]
    stream = torch.cuda.Stream()
    ctx = pic.Context(pic.make_config(w, capacity=cap, kernel=kernel), stream=stream)
    dev = [{k: v.cuda() for k, v in p.items()} for p in parts]
    EB = I.field_window(w, 2)[1].cuda()
    torch.cuda.synchronize()          # torch's copies before libpic's stream reads them
    for s, p in enumerate(dev):
        ctx.set_particles(s, p)
    ctx.set_fields(EB)
    ctx.set_graph(True)
    l0 = ctx.launch_count()
    for c in range(cycles):
        if c % 2 == 1:
            ctx.set_fields(EB)
        ctx.cycle()
    ctx.sync()
    assert ctx.launch_count() > l0
    for s, sp in enumerate(w.species):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        gm = ctx.get_moments(s).cpu().numpy()
        rep = {"species": sp.name}
        assert PU.compare_particles(w, sp, gp, orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(gm, orc[s][2], orc[s][3], rep), rep
    ctx.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_run_to_run_determinism(kernel):
    """SURVEY.md §5 (race detection): the mover is per-particle pure, so two runs
    of the same inputs give every particle (by id) bit for bit the same state,
    whatever order the atomics built; the moments differ only by the order of
    their fp64 sums."""
    w = I.c2(nx_per_rank=16, ppc=27)
    parts = I.make_species(w, device="cpu")
    a, _ = run_gpu(w, parts, 3, kernel)
    b, _ = run_gpu(w, parts, 3, kernel)
    for s in range(len(parts)):
        ga, gb = a[s][0], b[s][0]
        oa, ob = np.argsort(ga["id"]), np.argsort(gb["id"])
        assert np.array_equal(ga["id"][oa], gb["id"][ob])
        for k in "xyzuvwq":
            assert np.array_equal(ga[k][oa], gb[k][ob]), k
        ma, mb = a[s][1], b[s][1]
        scale = np.abs(ma).max(axis=(1, 2, 3), keepdims=True)
        assert np.all(np.abs(ma - mb) <= 1e-12 * scale)
