"""Host-side checks of the seeded input recipes, no GPU.

The generators hold none of the method's arithmetic; these tests pin the
workload structure the parity and bench runs rely on: particle counts per
cell, co-location of e-/p+ pairs, charge neutrality of a pair, the planet hole
and slab independence of the particle ids.
"""
import math

import torch

from paper_2507_20719_b200 import inputs as I


def test_uniform_ppc_counts_and_colocation():
    w = I.c1()
    e, p = I.make_species(w)
    assert e["x"].numel() == 16 ** 3 * 27
    assert torch.equal(e["x"], p["x"]) and torch.equal(e["z"], p["z"])
    # an e-/p+ pair is neutral cell by cell (equal |q|, opposite sign)
    assert torch.allclose(e["q"], -p["q"])
    # q_p = sign n0 V / ppc (R14)
    V = math.prod(w.delta)
    assert torch.allclose(p["q"], torch.full_like(p["q"], I.N0 * V / 27))


def test_c5_nonuniform_ppc_and_planet_hole():
    w = I.c5(ncell=(64, 32, 32), wind_ppc=4, inner_ppc=1, planet_ppc=32)
    parts = I.make_species(w)
    assert len(parts) == 4
    c, R = w.planet_center, w.planet_radius
    for d in parts:
        r2 = (d["x"] - c[0]) ** 2 + (d["y"] - c[1]) ** 2 + (d["z"] - c[2]) ** 2
        assert bool((r2 >= R * R).all())
    # wind pair co-located, planetary pair co-located, groups distinct
    assert torch.equal(parts[0]["x"], parts[1]["x"]) and torch.equal(parts[2]["y"], parts[3]["y"])
    assert parts[0]["x"].numel() != parts[2]["x"].numel()
    # non-uniform: the wind carries 1 ppc inside the ellipsoid, 4 outside; the
    # represented density is uniform, so q scales as 1/ppc
    q = parts[1]["q"]
    V = math.prod(w.delta)
    assert torch.allclose(torch.unique(q), torch.tensor([I.N0 * V / 4, I.N0 * V / 1], dtype=torch.float64))
    # planetary ppc decays away from the surface: more particles in the inner shell
    r = torch.sqrt((parts[2]["x"] - c[0]) ** 2 + (parts[2]["y"] - c[1]) ** 2 + (parts[2]["z"] - c[2]) ** 2)
    def per_volume(a, b):
        return int(((r >= a) & (r < b)).sum()) / (4 / 3 * math.pi * (b ** 3 - a ** 3))
    near, far = per_volume(R + 0.125, R + 0.25), per_volume(R + 0.5, R + 0.625)
    assert near > 2 * far > 0


def test_ids_independent_of_slab_split():
    w = I.c2(nx_per_rank=8, ppc=8, scale_x=2)
    full = I.make_species(w)[0]["id"]
    a = I.make_species(w.with_slab(0, 8))[0]["id"]
    b = I.make_species(w.with_slab(8, 16))[0]["id"]
    assert torch.equal(torch.sort(full).values, torch.sort(torch.cat([a, b])).values)


def test_plane_counts_match_generated_particles():
    """The per-x-plane histogram that count-balanced slabs cut (H10) agrees with
    the particles the generator draws (exactly away from the planet)."""
    w = I.c5(ncell=(64, 32, 32), wind_ppc=4, inner_ppc=1, planet_ppc=32)
    counts = I.plane_counts(w)
    parts = I.make_species(w)
    got = torch.zeros(w.ncell[0], dtype=torch.float64)
    for p in parts:
        cx = torch.floor(p["x"] / w.delta[0]).to(torch.int64)
        got.index_add_(0, cx, torch.ones_like(p["x"]))
    assert abs(float(got.sum()) - float(counts.sum())) < 0.02 * float(counts.sum())
    far = torch.arange(w.ncell[0]) < 20           # planes away from the moon
    assert torch.equal(got[far], counts[far])


def test_chunked_generation_matches_recipe():
    """The sub-slab generator of the full-size bench (C3-C5) draws the same
    particle set shape as one-piece generation: identical ids per cell, the
    slab, co-located e-/p+ pairs, the upper bound of `species_upper_counts`."""
    w = I.c5(ncell=(64, 32, 32), wind_ppc=4, inner_ppc=1, planet_ppc=32).with_slab(20, 44)
    ub = I.species_upper_counts(w)
    a = I.make_species_chunked(w, chunk_particles=20000)
    b = I.make_species(w)
    for s in range(len(w.species)):
        assert a[s]["x"].numel() <= ub[s]
        # ids encode (cell, in-cell index): per-cell counts agree except in cells the
        # moon cuts (positions are redrawn, so the cut differs)
        ca = torch.bincount((a[s]["id"] % (1 << 40)) // 1024, minlength=64 * 32 * 32)
        cb = torch.bincount((b[s]["id"] % (1 << 40)) // 1024, minlength=64 * 32 * 32)
        assert int((ca != cb).sum()) < 0.02 * int((cb > 0).sum())
        assert a[s]["id"].unique().numel() == a[s]["id"].numel()
        assert float(a[s]["x"].min()) >= 20 * w.delta[0] and float(a[s]["x"].max()) < 44 * w.delta[0]
    assert torch.equal(a[0]["x"], a[1]["x"]) and torch.equal(a[2]["z"], a[3]["z"])
