"""GPU edge cases with exact answers:

- P11 on the GPU: dyadic inputs (positions, velocities, charges on coarse
  dyadic grids, E = B = 0, Delta and dt powers of two) make every product and
  sum of Eq. 3 exact, so the GPU moments must equal the exact rational moments
  (Python fractions, no oracle) BIT FOR BIT in any summation order;
- R21 ties: particles that land exactly on cell, tile (4-cell) and slab faces
  and on the periodic boundary x = L are owned by the cell to the right, on one
  rank and across two loopback ranks, and match the oracle;
- R11: particles fast enough that a predictor-corrector iterate leaves the
  field window force the clamped sampling branch (stats.clamped > 0) of the
  tiled mover's global fallback; the final state matches the oracle's clamp.
"""
import dataclasses
from fractions import Fraction

import numpy as np
import pytest
import torch

import parity_util as PU
from paper_2507_20719_b200 import decomp, inputs as I, pic

pytestmark = pytest.mark.gpu
KERNELS = [pic.KERNEL_TILED, pic.KERNEL_BASIC]


def _zero_field_box(n=4, species=None):
    w = I.c1()
    sp = species or [dataclasses.replace(w.species[0]), dataclasses.replace(w.species[1])]
    return dataclasses.replace(w, name="dyadic", ncell=(n, n, n), length=(0.25 * n,) * 3, dt=0.5, species=sp,
                               field_params={"E": (0.0, 0.0, 0.0), "B": (0.0, 0.0, 0.0)})


def _run(w, parts, cycles, kernel):
    cap = [p["x"].numel() + 64 for p in parts]
    ctx = pic.Context(pic.make_config(w, capacity=cap, kernel=kernel))
    for s, p in enumerate(parts):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
    ctx.set_fields(I.field_window(w, 2)[1].cuda())
    for _ in range(cycles):
        ctx.cycle()
    stats = ctx.sync()
    out = [({k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}, ctx.get_moments(s).cpu().numpy())
           for s in range(len(parts))]
    ctx.close()
    return out, stats


def _exact_moments(w, parts, cycles):
    """Eq. 3 in exact rational arithmetic after `cycles` free-streaming steps
    (E = B = 0: v is unchanged and x advances by v dt, P1), periodic (R18)."""
    n = w.ncell
    d = [Fraction(w.length[k]) / n[k] for k in range(3)]
    V = d[0] * d[1] * d[2]
    L = [Fraction(w.length[k]) for k in range(3)]
    mom = np.zeros((10, n[2], n[1], n[0]))
    acc = {}
    for i in range(parts["x"].numel()):
        pos = [Fraction(float(parts[k][i])) for k in "xyz"]
        vel = [Fraction(float(parts[k][i])) for k in "uvw"]
        q = Fraction(float(parts["q"][i]))
        for _ in range(cycles):
            pos = [(pos[k] + vel[k] * Fraction(w.dt)) % L[k] for k in range(3)]
        xi = [pos[k] / d[k] for k in range(3)]
        c = [int(np.floor(float(xi[k]))) for k in range(3)]
        f = [xi[k] - c[k] for k in range(3)]
        vals = [1, vel[0], vel[1], vel[2], vel[0] * vel[0], vel[0] * vel[1], vel[0] * vel[2], vel[1] * vel[1],
                vel[1] * vel[2], vel[2] * vel[2]]
        for corner in range(8):
            b = [(corner >> k) & 1 for k in range(3)]
            S = Fraction(1)
            for k in range(3):
                S *= f[k] if b[k] else 1 - f[k]
            node = tuple((c[k] + b[k]) % n[k] for k in range(3))
            for m in range(10):
                acc[(m,) + node] = acc.get((m,) + node, Fraction(0)) + q * S * vals[m] / V
    for (m, x, y, z), v in acc.items():
        mom[m, z, y, x] = float(v)
        assert Fraction(mom[m, z, y, x]) == v, "expected value not representable: bad test input"
    return mom


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_p11_dyadic_moments_bit_exact(kernel, seed):
    w = _zero_field_box()
    rng = np.random.default_rng(seed)
    parts = []
    for s in range(2):
        k = int(rng.integers(1, 9))
        # positions on a 1/64-cell grid, velocities on 1/16 multiples of a
        # power of two (|v dt| < 2 cells), charges +-j/8
        pos = rng.integers(0, 4 * 64, size=(3, k)) / 64.0 * 0.25
        vel = rng.integers(-32, 33, size=(3, k)) / 16.0 * 0.0625
        q = (rng.integers(1, 9, size=k) / 8.0) * (1 if s else -1)
        parts.append({"x": torch.tensor(pos[0]), "y": torch.tensor(pos[1]), "z": torch.tensor(pos[2]),
                      "u": torch.tensor(vel[0]), "v": torch.tensor(vel[1]), "w": torch.tensor(vel[2]),
                      "q": torch.tensor(q), "id": torch.arange(k, dtype=torch.int64) + 100 * s})
    cycles = 2
    out, stats = _run(w, parts, cycles, kernel)
    assert stats["nonfinite"] == 0 and stats["clamped"] == 0
    for s in range(2):
        want = _exact_moments(w, parts[s], cycles)
        got = out[s][1]
        assert got.shape == want.shape
        assert np.array_equal(got, want), np.argwhere(got != want)[:5]


def _face_particles(w, s):
    """Particles that land exactly on faces after one free-streaming step
    (dt = 0.5, Delta = 0.25): x^n on a quarter-cell grid, v dt a whole number
    of quarter cells, so x^{n+1} is exact."""
    d = w.delta[0]
    L = w.length[0]
    # (x^n, v) pairs along x; y, z mid-cell
    cases = [
        (3.5 * d, 0.5 * d / w.dt),        # -> 4.0: tile face (4-cell tiles), slab face of P = 4
        (7.75 * d, 0.25 * d / w.dt),      # -> 8.0: slab face of P = 2 (tie goes right, R21)
        (8.25 * d, -0.25 * d / w.dt),     # -> 8.0 from the right
        (L - 0.5 * d, 0.5 * d / w.dt),    # -> L: periodic wrap to exactly 0 (R10)
        (0.5 * d, -0.5 * d / w.dt),       # -> 0.0 from the right
        (1.5 * d, -1.5 * d / w.dt),       # -> 0.0
        (5.0 * d, 0.0),                   # stays on a cell face
        (12.0 * d, 1.0 * d / w.dt),       # node to node: 12 -> 13
    ]
    n = len(cases)
    x = torch.tensor([c[0] for c in cases], dtype=torch.float64)
    u = torch.tensor([c[1] for c in cases], dtype=torch.float64)
    y = torch.full((n,), 2.5 * d, dtype=torch.float64) + 0.25 * d * torch.arange(n)
    z = torch.full((n,), 6.0 * d, dtype=torch.float64)     # on a y-z node plane too
    return {"x": x, "y": y, "z": z, "u": u, "v": torch.zeros(n, dtype=torch.float64),
            "w": torch.zeros(n, dtype=torch.float64), "q": torch.full((n,), 0.125 * (1 if s else -1), dtype=torch.float64),
            "id": torch.arange(n, dtype=torch.int64) + 1000 * s}


@pytest.mark.parametrize("kernel", KERNELS)
def test_r21_face_ties_one_rank(kernel):
    w = _zero_field_box(n=16)
    parts = [_face_particles(w, s) for s in range(2)]
    orc = PU.run_oracle(w, parts, 1)
    out, stats = _run(w, parts, 1, kernel)
    for s, sp in enumerate(w.species):
        rep = {}
        assert PU.compare_particles(w, sp, out[s][0], orc[s][0], orc[s][1], rep), rep
        assert rep["pos_ratio"] == 0.0            # exact: every landing point is dyadic
        assert np.array_equal(out[s][1], orc[s][2])   # one particle per node set: exact
    gx = out[0][0]["x"]
    assert np.count_nonzero(gx == 0.0) == 3 and np.count_nonzero(gx == 2.0) == 2


def test_r21_face_ties_across_loopback_slabs():
    """The particles landing on x = 8 Delta (the P = 2 slab face) must end on
    rank 1, those landing on x = L (= 0) on rank 0."""
    import slab_parity as SP
    from test_gpu_loopback import run_loopback
    w = _zero_field_box(n=16)

    def make(_w, device="cpu"):
        return [_face_particles(w, s) for s in range(2)]
    orig = I.make_species
    I.make_species = make
    try:
        gathered, parts_all = run_loopback(w, 1, 2, pic.KERNEL_TILED, sources=False)
    finally:
        I.make_species = orig
    orc = PU.run_oracle(w, parts_all, 1)
    ok, reps = SP.check_union("faces", w, gathered, orc, kernel=pic.KERNEL_TILED, transport="loopback", world=2)
    assert ok, reps
    x1 = gathered[1][0][0][0]["x"]
    x0 = gathered[0][0][0][0]["x"]
    d = w.delta[0]
    assert np.count_nonzero(x1 == 8 * d) == 2 and np.count_nonzero(x0 == 8 * d) == 0
    assert np.count_nonzero(x0 == 0.0) == 3


@pytest.mark.parametrize("kernel", KERNELS)
def test_r11_clamped_samples_match_the_oracle(kernel):
    """|v| dt/2 = 6 cells > the G = 2 ghost nodes: the iterates after the first
    sample outside the field window (clamped to it on both sides, R11)."""
    w = I.c1(randomized=True)
    parts = I.make_species(w, device="cpu")
    fast = []
    dirs = [(1, 0, 0), (0, -1, 0), (0, 0, 1), (-1, 1, 1), (1, -1, -1)]
    for s, p in enumerate(parts):
        n = len(dirs)
        speed = 6 * w.delta[0] / (w.dt / 2) / np.sqrt(3)
        vel = torch.tensor(dirs, dtype=torch.float64) * speed
        extra = {"x": torch.full((n,), 0.6 * w.delta[0]) + 0.1 * torch.arange(n) * w.delta[0],
                 "y": torch.full((n,), 15.4 * w.delta[1]), "z": torch.full((n,), 1.3 * w.delta[2]),
                 "u": vel[:, 0].contiguous(), "v": vel[:, 1].contiguous(), "w": vel[:, 2].contiguous(),
                 "q": p["q"][:n].clone(), "id": torch.arange(n, dtype=torch.int64) + (1 << 50)}
        fast.append({k: torch.cat([p[k], extra[k]]).contiguous() for k in p})
    orc = PU.run_oracle(w, fast, 2)
    out, stats = _run(w, fast, 2, kernel)
    assert stats["clamped"] > 0, stats
    for s, sp in enumerate(w.species):
        rep = {}
        assert PU.compare_particles(w, sp, out[s][0], orc[s][0], orc[s][1], rep), rep
        assert PU.compare_moments(out[s][1], orc[s][2], orc[s][3], rep), rep
