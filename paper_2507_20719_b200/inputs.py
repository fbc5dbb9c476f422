"""Seeded synthetic inputs for the particle hot path (configs C1..C5).

This module is the ONLY code shared by the oracle tests and the CUDA path: it
draws particles and evaluates analytic fields at grid nodes.  It holds none of
the method's arithmetic (no mover, no interpolation, no deposit).  Every
workload is a `Workload` recipe; `make_species` / `field_window` turn it into
torch tensors on any device (CPU for the oracle-sized cases, CUDA for the full
sizes).  Recipes follow SURVEY.md §8(d) d.1 and DESIGN.md §5:

  code units: c = 1, lengths in d_i, time in 1/omega_pi,
  q/m_i = +1, n0 = 1/(4 pi) so omega_pi = 1; q_p = sign * n(x) V / ppc.

C1  16^3 periodic uniform Maxwellian, e-/p+, 27 ppc, uniform E x B (C1r: the
    same with per-node +-10 % random fields so gather-index bugs show).
C2  GEM-style double Harris sheet, 128 x 64 x 32, 125 ppc, m_i/m_e = 256,
    q_p proportional to n(y) ("inspired by the GEM challenge").
C3  weak-scaling cube, 192^3 cells per GPU, 64 ppc, B0 z + random Fourier modes.
C4  Mercury-like open-boundary dipole magnetosphere with drifting solar wind.
C5  Ganymede-like 4-species magnetosphere with strongly non-uniform ppc.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import torch

PERIODIC, OPEN = 0, 1
N0 = 1.0 / (4.0 * math.pi)


@dataclass
class Species:
    name: str
    qom: float                      # q_s / m_s (signed)
    sign: float                     # sign of q_s
    vth: float                      # thermal speed per component
    drift: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    ppc: int = 27
    # optional non-uniform loading (C5): ppc_fn(Xc, Yc, Zc) -> int64 particles per
    # cell at the cell centres, dens_fn(X, Y, Z) -> number density at positions;
    # species of one `group` share positions (co-located pairs)
    ppc_fn: Optional[Callable] = None
    dens_fn: Optional[Callable] = None
    group: int = 0


@dataclass
class Workload:
    name: str
    ncell: Tuple[int, int, int]
    length: Tuple[float, float, float]
    bc: Tuple[int, int, int]
    dt: float
    species: List[Species]
    n_iter: int = 3
    c: float = 1.0
    cycles: int = 5
    seed: int = 1
    # fields: callable (X, Y, Z tensors of node positions, float64) -> 6 tensors
    fields: Optional[Callable] = None
    field_kind: str = "uniform"
    field_params: dict = field(default_factory=dict)
    planet_center: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    planet_radius: float = 0.0
    colocate: bool = True           # e-/p+ pairs at the same positions
    density: str = "uniform"        # or "harris"
    slab: Tuple[int, int] = (0, 0)  # x-cells [lo, hi) of this rank (set by with_slab)
    relativistic: bool = False      # Eq. 2 with gamma (NEXT-1)

    @property
    def delta(self):
        return tuple(self.length[d] / self.ncell[d] for d in range(3))

    def with_slab(self, lo: int, hi: int) -> "Workload":
        import copy
        w = copy.copy(self)
        w.slab = (lo, hi)
        return w

    def slab_or_all(self):
        return self.slab if self.slab[1] > self.slab[0] else (0, self.ncell[0])


# ------------------------------------------------------------------ fields --
def _uniform(E, B):
    def fn(X, Y, Z, w):
        one = torch.ones_like(X)
        return [E[0] * one, E[1] * one, E[2] * one, B[0] * one, B[1] * one, B[2] * one]
    return fn


def _harris_fields(X, Y, Z, w: Workload):
    p = w.field_params
    B0, lam, psi0 = p["B0"], p["lam"], p["psi0"]
    Lx, Ly = w.length[0], w.length[1]
    y1, y2 = Ly / 4, 3 * Ly / 4
    Bx = B0 * (torch.tanh((Y - y1) / lam) - torch.tanh((Y - y2) / lam) - 1.0)
    # GEM perturbation psi = psi0 cos(2 pi x / Lx) cos(4 pi y / Ly) (periodic in y)
    kx, ky = 2 * math.pi / Lx, 4 * math.pi / Ly
    Bx = Bx + psi0 * ky * torch.cos(kx * X) * torch.sin(ky * Y)
    By = -psi0 * kx * torch.sin(kx * X) * torch.cos(ky * Y)
    zero = torch.zeros_like(X)
    return [zero, zero, zero, Bx, By, zero]


def _fourier_fields(X, Y, Z, w: Workload):
    """B0 z + 4 random Fourier modes per component (10 %), E = v_E background + modes."""
    p = w.field_params
    B0, E0 = p["B0"], p["E0"]
    g = torch.Generator().manual_seed(1000 + w.seed)
    L = w.length_global if hasattr(w, "length_global") else w.length
    out = [E0[0] + 0 * X, E0[1] + 0 * X, E0[2] + 0 * X, 0 * X, 0 * X, B0 + 0 * X]
    scales = [0.1 * max(abs(e) for e in E0) or 1e-6] * 3 + [0.1 * B0] * 3
    for comp in range(6):
        for _ in range(4):
            k = torch.randint(1, 4, (3,), generator=g).tolist()
            ph = torch.rand(3, generator=g).tolist()
            amp = scales[comp] * (torch.rand(1, generator=g).item() - 0.5) * 0.5
            out[comp] = out[comp] + amp * (torch.cos(2 * math.pi * (k[0] * X / L[0] + ph[0]))
                                           * torch.cos(2 * math.pi * (k[1] * Y / L[1] + ph[1]))
                                           * torch.cos(2 * math.pi * (k[2] * Z / L[2] + ph[2])))
    return out


def _dipole_fields(X, Y, Z, w: Workload):
    """Point dipole M || -z at the planet centre + IMF; E = -v_sw x B_IMF / c.
    The dipole is clamped inside the planet radius (field of the surface)."""
    p = w.field_params
    cx, cy, cz = w.planet_center
    M, Bimf, vsw = p["M"], p["Bimf"], p["vsw"]
    dx, dy, dz = X - cx, Y - cy, Z - cz
    r = torch.sqrt(dx * dx + dy * dy + dz * dz).clamp_min(w.planet_radius)
    mz = -M
    # B = (3 (m.r) r / r^5 - m / r^3)
    mdotr = mz * dz
    r5 = r ** 5
    r3 = r ** 3
    Bx = 3 * mdotr * dx / r5 + Bimf[0]
    By = 3 * mdotr * dy / r5 + Bimf[1]
    Bz = 3 * mdotr * dz / r5 - mz / r3 + Bimf[2]
    v = (vsw, 0.0, 0.0)
    Ex = -(v[1] * Bimf[2] - v[2] * Bimf[1]) / w.c + 0 * X
    Ey = -(v[2] * Bimf[0] - v[0] * Bimf[2]) / w.c + 0 * X
    Ez = -(v[0] * Bimf[1] - v[1] * Bimf[0]) / w.c + 0 * X
    return [Ex, Ey, Ez, Bx, By, Bz]


def node_field_values(w: Workload, lo: Sequence[int], n: Sequence[int], device="cpu") -> torch.Tensor:
    """EB[kz][ky][kx][6] at global node indices [lo_d, lo_d + n_d); periodic axes
    map node g to position (g mod N) Delta (replicated images), open axes to g Delta."""
    dl = w.delta
    coords = []
    for d in range(3):
        g = torch.arange(lo[d], lo[d] + n[d], dtype=torch.int64, device=device)
        if w.bc[d] == PERIODIC:
            g = torch.remainder(g, w.ncell[d])
        coords.append(g.to(torch.float64) * dl[d])
    Z, Y, X = torch.meshgrid(coords[2], coords[1], coords[0], indexing="ij")
    if w.field_kind == "uniform":
        vals = _uniform(w.field_params["E"], w.field_params["B"])(X, Y, Z, w)
    elif w.field_kind == "harris":
        vals = _harris_fields(X, Y, Z, w)
    elif w.field_kind == "fourier":
        vals = _fourier_fields(X, Y, Z, w)
    elif w.field_kind == "dipole":
        vals = _dipole_fields(X, Y, Z, w)
    else:
        raise ValueError(w.field_kind)
    EB = torch.stack(vals, dim=-1).contiguous()
    rel = w.field_params.get("random_rel", 0.0)
    if rel:
        # per unique node +-rel * |reference| perturbation, keyed by the
        # unique (periodic-wrapped) node index so images stay consistent
        gen = torch.Generator().manual_seed(4242 + w.seed)
        uniq = [w.ncell[d] if w.bc[d] == PERIODIC else w.ncell[d] + 2 * 8 + 1 for d in range(3)]
        noise = (torch.rand((uniq[2], uniq[1], uniq[0], 6), generator=gen, dtype=torch.float64) * 2 - 1)
        ref = torch.tensor([max(map(abs, w.field_params["E"]))] * 3 + [max(map(abs, w.field_params["B"]))] * 3,
                           dtype=torch.float64)
        idx = []
        for d in range(3):
            g = torch.arange(lo[d], lo[d] + n[d], dtype=torch.int64)
            g = torch.remainder(g, w.ncell[d]) if w.bc[d] == PERIODIC else (g + 8).clamp(0, uniq[d] - 1)
            idx.append(g)
        pert = noise[idx[2]][:, idx[1]][:, :, idx[0]] * (rel * ref)
        EB = EB + pert.to(device)
    return EB


def window_bounds(w: Workload, ghost: int):
    """Global node box of the field window of this rank (pic.h pic_set_fields)."""
    lo_x, hi_x = w.slab_or_all()
    lo = (lo_x - ghost, -ghost, -ghost)
    n = (hi_x - lo_x + 1 + 2 * ghost, w.ncell[1] + 1 + 2 * ghost, w.ncell[2] + 1 + 2 * ghost)
    return lo, n


def field_window(w: Workload, ghost: int, device="cpu") -> Tuple[Tuple[int, int, int], torch.Tensor]:
    lo, n = window_bounds(w, ghost)
    return lo, node_field_values(w, lo, n, device=device)


# --------------------------------------------------------------- particles --
def _density(w: Workload, y: torch.Tensor) -> torch.Tensor:
    if w.density == "uniform":
        return torch.full_like(y, N0)
    p = w.field_params
    Ly, lam, nb = w.length[1], p["lam"], p["nb"]
    y1, y2 = Ly / 4, 3 * Ly / 4
    return N0 * (1.0 / torch.cosh((y - y1) / lam) ** 2 + 1.0 / torch.cosh((y - y2) / lam) ** 2 + nb)


def _sheet_fraction(w: Workload, y: torch.Tensor):
    p = w.field_params
    Ly, lam, nb = w.length[1], p["lam"], p["nb"]
    y1, y2 = Ly / 4, 3 * Ly / 4
    s1 = 1.0 / torch.cosh((y - y1) / lam) ** 2
    s2 = 1.0 / torch.cosh((y - y2) / lam) ** 2
    tot = s1 + s2 + nb
    return s1 / tot, s2 / tot


def cell_range(w: Workload):
    lo, hi = w.slab_or_all()
    return lo, hi


def _cell_centres(w: Workload, device):
    lo, hi = cell_range(w)
    nx, ny, nz = hi - lo, w.ncell[1], w.ncell[2]
    c = torch.arange(nx * ny * nz, device=device, dtype=torch.int64)
    cx, cy, cz = c % nx + lo, (c // nx) % ny, c // (nx * ny)
    dl = w.delta
    return cx, cy, cz, ((cx.double() + 0.5) * dl[0], (cy.double() + 0.5) * dl[1], (cz.double() + 0.5) * dl[2])


def make_positions(w: Workload, sp: Species, gen: torch.Generator, device, planet_ok=True):
    """Particles uniformly random in every cell of this rank's slab: sp.ppc per
    cell, or sp.ppc_fn(cell centre) for non-uniform loading.  ids = global cell
    id * 1024 + in-cell index, independent of the slab split."""
    cx, cy, cz, cen = _cell_centres(w, device)
    if sp.ppc_fn is not None:
        counts = sp.ppc_fn(*cen).to(torch.int64).clamp(0, 1023)
    else:
        counts = torch.full_like(cx, sp.ppc)
    n = int(counts.sum().item())
    cell = torch.repeat_interleave(torch.arange(cx.numel(), device=device), counts)
    start = torch.cumsum(counts, 0) - counts
    k = torch.arange(n, device=device, dtype=torch.int64) - start[cell]
    cx, cy, cz = cx[cell], cy[cell], cz[cell]
    dl = w.delta
    r = torch.rand((3, n), generator=gen, device=device, dtype=torch.float64)
    x = (cx.to(torch.float64) + r[0]) * dl[0]
    y = (cy.to(torch.float64) + r[1]) * dl[1]
    z = (cz.to(torch.float64) + r[2]) * dl[2]
    gid = ((cz * w.ncell[1] + cy) * w.ncell[0] + cx) * 1024 + k
    keep = None
    if w.planet_radius > 0 and planet_ok:
        c = w.planet_center
        keep = ((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) >= w.planet_radius ** 2
    return x, y, z, gid, keep, counts[cell]


def plane_counts(w: Workload, device="cpu") -> torch.Tensor:
    """Expected particles per global x-plane of cells (all species; the planet
    volume counted as empty): the histogram that count-balanced slabs cut
    (SURVEY.md H10).  Uses the species' ppc at the cell centres."""
    full = w.with_slab(0, w.ncell[0])
    cx, cy, cz, cen = _cell_centres(full, device)
    tot = torch.zeros(w.ncell[0], dtype=torch.float64, device=device)
    keep = torch.ones_like(cx, dtype=torch.bool)
    if w.planet_radius > 0:
        c = w.planet_center
        keep = ((cen[0] - c[0]) ** 2 + (cen[1] - c[1]) ** 2 + (cen[2] - c[2]) ** 2) >= w.planet_radius ** 2
    for sp in w.species:
        n = sp.ppc_fn(*cen).to(torch.float64) if sp.ppc_fn is not None else torch.full_like(cx, sp.ppc, dtype=torch.float64)
        tot.index_add_(0, cx, n * keep)
    return tot


def make_species(w: Workload, device="cpu") -> List[dict]:
    """Particles of every species of this rank: list of dicts of float64 tensors
    x y z u v w q and int64 id (global: cell id * 1024 + in-cell index, plus
    species * 2^40).  q_p = sign * n(x) V / ppc_cell (R14)."""
    gen = torch.Generator(device=device).manual_seed(w.seed * 7919 + w.slab_or_all()[0])
    out = []
    groups = {}
    V = w.delta[0] * w.delta[1] * w.delta[2]
    for si, sp in enumerate(w.species):
        key = sp.group if w.colocate else si
        if key not in groups:
            groups[key] = make_positions(w, sp, gen, device)
        x, y, z, gid, keep, ppc_cell = groups[key]
        n = x.numel()
        dens = sp.dens_fn(x, y, z) if sp.dens_fn is not None else _density(w, y)
        q = sp.sign * dens * V / ppc_cell.to(torch.float64)
        vel = torch.randn((3, n), generator=gen, device=device, dtype=torch.float64) * sp.vth
        if w.relativistic:
            # draw the momentum per unit mass u = gamma v, so |v| = |u| / sqrt(1 + u^2/c^2) < c
            vel = vel / torch.sqrt(1.0 + (vel * vel).sum(0, keepdim=True) / (w.c * w.c))
        u, v, ww = vel[0] + sp.drift[0], vel[1] + sp.drift[1], vel[2] + sp.drift[2]
        if w.density == "harris":
            # sheet populations drift along +-z (GEM); background is at rest
            f1, f2 = _sheet_fraction(w, y)
            pick = torch.rand(n, generator=gen, device=device, dtype=torch.float64)
            vd = w.field_params["vd_i"] if sp.sign > 0 else w.field_params["vd_e"]
            ww = ww + torch.where(pick < f1, vd, torch.where(pick < f1 + f2, -vd, 0.0))
        d = {"x": x.clone(), "y": y.clone(), "z": z.clone(), "u": u.contiguous(), "v": v.contiguous(),
             "w": ww.contiguous(), "q": q.contiguous(), "id": gid.clone() + si * (1 << 40)}
        if keep is not None:
            d = {k: t[keep].contiguous() for k, t in d.items()}
        out.append(d)
    return out


def species_upper_counts(w: Workload) -> List[int]:
    """Particles per species of this rank's slab before the planet cut (an upper
    bound of `make_species`' counts): the capacity of a store allocated before
    the particles are drawn."""
    cx, cy, cz, cen = _cell_centres(w, "cpu")
    out = []
    for sp in w.species:
        if sp.ppc_fn is not None:
            out.append(int(sp.ppc_fn(*cen).to(torch.int64).clamp(0, 1023).sum().item()))
        else:
            out.append(int(cx.numel()) * sp.ppc)
    return out


def iter_species_chunks(w: Workload, chunk_particles: int = 64_000_000, device="cpu"):
    """Yield `make_species` of consecutive sub-slabs of whole x-planes of this
    rank's slab (each seeded by its first plane, as `make_species` seeds a
    slab), about `chunk_particles` particles per sub-slab: the particles of a
    slab too large to draw in one piece (C3-C5 at full size), to be appended to
    a store one sub-slab at a time (pic_add_particles).  Yields (lo, hi, parts)."""
    lo, hi = w.slab_or_all()
    ub = species_upper_counts(w)
    step = max(1, int(chunk_particles * (hi - lo) // max(1, sum(ub))))
    for a in range(lo, hi, step):
        b = min(hi, a + step)
        yield a, b, make_species(w.with_slab(a, b), device=device)


def make_species_chunked(w: Workload, chunk_particles: int = 32_000_000) -> List[dict]:
    """`make_species` for slabs too large to draw in one piece (C3-C5 at full
    size): the slab is drawn in sub-slabs of whole x-planes (each seeded by its
    first plane, as `make_species` seeds a slab) and assembled in host memory,
    so the transient memory is one sub-slab's.  Same recipe and co-location;
    a different random stream from a one-piece draw of the same slab."""
    lo, hi = w.slab_or_all()
    ub = species_upper_counts(w)
    step = max(1, int(chunk_particles * (hi - lo) // max(1, sum(ub))))
    keys = ("x", "y", "z", "u", "v", "w", "q", "id")
    out = [{k: torch.empty(ub[s], dtype=torch.int64 if k == "id" else torch.float64) for k in keys}
           for s in range(len(w.species))]
    fill = [0] * len(w.species)
    for a in range(lo, hi, step):
        parts = make_species(w.with_slab(a, min(hi, a + step)), device="cpu")
        for s, p in enumerate(parts):
            n = p["x"].numel()
            for k in keys:
                out[s][k][fill[s]:fill[s] + n].copy_(p[k])
            fill[s] += n
        del parts
    return [{k: t[:fill[s]] for k, t in out[s].items()} for s in range(len(w.species))]


# ----------------------------------------------------------------- configs --
def c1(randomized: bool = False, seed: int = 1) -> Workload:
    fp = {"E": (0.0, 1e-4, 0.0), "B": (0.0, 0.0, 0.01)}
    if randomized:
        fp["random_rel"] = 0.1
    return Workload(
        name="c1r" if randomized else "c1", ncell=(16, 16, 16), length=(4.0, 4.0, 4.0),
        bc=(PERIODIC,) * 3, dt=0.5, seed=seed,
        species=[Species("e-", -256.0, -1.0, 0.05, ppc=27), Species("p+", 1.0, 1.0, 0.0070, ppc=27)],
        field_kind="uniform", field_params=fp)


def c1rel(seed: int = 6) -> Workload:
    """NEXT-1 check: C1 with relativistic thermal speeds (electron v_th = 0.3 c, so
    gamma up to ~2 in the tail; v drawn below c) and the relativistic mover."""
    w = c1(randomized=True, seed=seed)
    w.relativistic = True
    w.species[0].vth = 0.3
    w.species[1].vth = 0.05
    w.field_params = dict(w.field_params, B=(0.0, 0.0, 0.05))
    return w


def c2(scale_x: int = 1, nx_per_rank: int = 128, seed: int = 2, ppc: int = 125) -> Workload:
    """GEM Harris: 128 x 64 x 32 cells per rank along x (weak-scaled by scale_x ranks)."""
    B0 = 0.0195
    Te = B0 * B0 / 12.0
    vthe, vthi = math.sqrt(256.0 * Te), math.sqrt(5.0 * Te)
    vdi = 20.0 * Te / B0
    fp = {"B0": B0, "lam": 0.5, "nb": 0.2, "psi0": 0.1 * B0, "vd_i": vdi, "vd_e": -vdi / 5.0}
    nx = nx_per_rank * scale_x
    return Workload(
        name="c2", ncell=(nx, 64, 32), length=(0.2 * nx, 12.8, 6.4), bc=(PERIODIC,) * 3, dt=0.125,
        seed=seed, species=[Species("e-", -256.0, -1.0, vthe, ppc=ppc), Species("p+", 1.0, 1.0, vthi, ppc=ppc)],
        field_kind="harris", field_params=fp, density="harris")


def c3(nranks: int = 1, n_per_rank: int = 192, ppc: int = 64, seed: int = 3) -> Workload:
    nx = n_per_rank * nranks
    w = Workload(
        name="c3", ncell=(nx, n_per_rank, n_per_rank), length=(0.25 * nx, 0.25 * n_per_rank, 0.25 * n_per_rank),
        bc=(PERIODIC,) * 3, dt=0.5, seed=seed,
        species=[Species("e-", -256.0, -1.0, 0.05, ppc=ppc), Species("p+", 1.0, 1.0, 0.0070, ppc=ppc)],
        field_kind="fourier", field_params={"B0": 0.01, "E0": (0.0, 1e-4, 0.0)})
    return w


def c4(ncell=(512, 256, 256), ppc: int = 64, seed: int = 4) -> Workload:
    """Open-boundary dipole magnetosphere; lengths scale with the cell count at Delta = 0.125."""
    d = 0.125
    L = tuple(n * d for n in ncell)
    center = (L[0] * 24 / 64, L[1] / 2, L[2] / 2)
    R = 2.0 * ncell[0] / 512
    vsw = 0.02
    # standoff ~ 6 d_i (scaled): pressure balance B^2/(8 pi) ~ n m v^2
    M = 0.005 * (6.0 * ncell[0] / 512) ** 3 * 8
    return Workload(
        name="c4", ncell=ncell, length=L, bc=(OPEN,) * 3, dt=0.25, seed=seed,
        species=[Species("e-", -256.0, -1.0, 0.05, (vsw, 0, 0), ppc=ppc),
                 Species("p+", 1.0, 1.0, 0.0031, (vsw, 0, 0), ppc=ppc)],
        field_kind="dipole", field_params={"M": M, "Bimf": (0.0, 0.0, -0.005), "vsw": vsw},
        planet_center=center, planet_radius=R)


def c5(ncell=(512, 256, 256), wind_ppc: int = 64, inner_ppc: int = 8, planet_ppc: int = 256, seed: int = 5) -> Workload:
    """Ganymede-like magnetosphere: 4 species (solar-wind e-/p+ in a sub-Alfvenic
    flow, planetary e-/p+ from the moon's surface), open boundaries, absorbing
    moon, strongly non-uniform ppc: wind 64 ppc outside a magnetosphere
    ellipsoid and 8 inside, planetary round(256 exp(-(r - R)/2)) (0..256).
    Densities are smooth (weights carry n(x)), so ppc and weights vary, not n."""
    d = 0.125
    L = tuple(n * d for n in ncell)
    sc = ncell[0] / 512
    R = 2.0 * sc
    center = (L[0] * 0.5, L[1] / 2, L[2] / 2)
    vflow = 0.01
    M = 0.005 * (4.0 * sc) ** 3 * 8
    ax = (8.0 * sc, 6.0 * sc, 6.0 * sc)    # magnetosphere ellipsoid semi-axes

    def r_of(X, Y, Z):
        return torch.sqrt((X - center[0]) ** 2 + (Y - center[1]) ** 2 + (Z - center[2]) ** 2)

    def wind_ppc_fn(X, Y, Z):
        inside = ((X - center[0]) / ax[0]) ** 2 + ((Y - center[1]) / ax[1]) ** 2 + ((Z - center[2]) / ax[2]) ** 2 < 1
        return torch.where(inside, inner_ppc, wind_ppc)

    def planet_ppc_fn(X, Y, Z):
        r = r_of(X, Y, Z)
        return torch.where(r >= R, torch.round(planet_ppc * torch.exp(-(r - R) / (2.0 * sc))), 0.0)

    def planet_dens(X, Y, Z):
        return 2.0 * N0 * torch.exp(-(r_of(X, Y, Z) - R) / (2.0 * sc))

    wind = lambda X, Y, Z: N0 + 0 * X
    return Workload(
        name="c5", ncell=ncell, length=L, bc=(OPEN,) * 3, dt=0.25, seed=seed,
        species=[Species("sw e-", -256.0, -1.0, 0.05, (vflow, 0, 0), ppc_fn=wind_ppc_fn, dens_fn=wind, group=0),
                 Species("sw p+", 1.0, 1.0, 0.0031, (vflow, 0, 0), ppc_fn=wind_ppc_fn, dens_fn=wind, group=0),
                 Species("pl e-", -256.0, -1.0, 0.02, ppc_fn=planet_ppc_fn, dens_fn=planet_dens, group=1),
                 Species("pl p+", 1.0, 1.0, 0.0015, ppc_fn=planet_ppc_fn, dens_fn=planet_dens, group=1)],
        field_kind="dipole", field_params={"M": M, "Bimf": (0.0, 0.0, -0.005), "vsw": vflow},
        planet_center=center, planet_radius=R)


CONFIGS = {"c1": c1, "c1r": lambda: c1(True), "c1rel": c1rel, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
