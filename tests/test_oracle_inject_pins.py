"""Pins of the NEXT-3 inflow injection oracle (reading R28 of
DESIGN.md §3), no GPU.

The random numbers come from Philox4x32-10, pinned to its published
known-answer vectors.  The injection itself is pinned by physics that does not
depend on the oracle's own code: with E = B = 0 a ghost particle enters iff it
crosses x = 0 during the step and moves by exactly v dt; the entered count of a
drifting Maxwellian matches the expected slab flux; velocities of a beam that
enters completely have the drawn mean and spread.
"""
import math

import numpy as np

import oracle as O
from test_oracle_pins import const_field, window

NC, LEN = (16, 8, 8), (4.0, 2.0, 2.0)      # Delta = 0.25
OPEN_X = (1, 0, 0)


def test_philox_known_answers():
    """Random123 known-answer vectors for philox4x32-10."""
    assert O.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def _field(g):
    return window(NC, 2, const_field((0, 0, 0), (0, 0, 0)), LEN)


def test_cold_beam_enters_by_crossing():
    """vth = 0, E = B = 0: the kept particles are exactly the ghost particles
    with x_old + v_d dt >= 0, each moved by v_d dt (y, z, v unchanged)."""
    dt, vd, ppc, seed, cyc = 0.5, 0.2, 16, 12345, 3
    g = O.make_grid(NC, LEN, bc=OPEN_X, dt=dt)
    inj = O.inject(g, _field(g), 1, 1.0, 3, seed, cyc, ppc, 0.0, (vd, 0, 0), 0.01)
    d = LEN[0] / NC[0]
    # regenerate the ghost positions from the (pinned) generator: call 0 -> x, y
    want = 0
    for gc in range(NC[1] * NC[2]):
        for k in range(ppc):
            c = O.philox([gc, k, cyc, (1 << 8) | 0], [seed & 0xFFFFFFFF, seed >> 32])
            u0 = ((c[0] >> 5) * 67108864.0 + (c[1] >> 6)) / 9007199254740992.0
            want += ((-1.0 + u0) * d + vd * dt) >= 0.0
    assert len(inj["x"]) == want
    assert np.all(inj["x"] >= 0) and np.all(inj["x"] <= vd * dt + 1e-15)
    np.testing.assert_array_equal(inj["u"], vd)
    assert not inj["v"].any() and not inj["w"].any()
    assert np.all(inj["q"] == 0.01)
    # ids unique and tagged
    assert len(np.unique(inj["id"])) == len(inj["id"]) and np.all(inj["id"] >> 62 == 1)


def test_warm_flux_matches_slab_expectation():
    """Entries per ghost particle = E[clip(v dt / dx, 0, 1)], v ~ N(vd, vth^2),
    integrated numerically here; the count must agree within 5 sigma."""
    dt, vd, vth, ppc = 0.5, 0.1, 0.2, 64
    g = O.make_grid(NC, LEN, bc=OPEN_X, dt=dt)
    inj = O.inject(g, _field(g), 0, -4.0, 3, 99, 0, ppc, vth, (vd, 0, 0), -0.01)
    d = LEN[0] / NC[0]
    v = np.linspace(vd - 10 * vth, vd + 10 * vth, 200001)
    pdf = np.exp(-0.5 * ((v - vd) / vth) ** 2) / (vth * math.sqrt(2 * math.pi))
    p = np.trapezoid(np.clip(v * dt / d, 0, 1) * pdf, v)
    n = NC[1] * NC[2] * ppc
    mean, sd = n * p, math.sqrt(n * p * (1 - p))
    assert abs(len(inj["x"]) - mean) < 5 * sd


def test_beam_that_fully_enters_has_the_drawn_distribution():
    """vd dt >= 2 dx and vth small: every ghost particle enters; with E = B = 0
    the kept velocities are the drawn ones: mean vd, std vth per component."""
    dt, vd, vth, ppc = 0.5, 1.0, 0.05, 64
    g = O.make_grid(NC, LEN, bc=OPEN_X, dt=dt)
    inj = O.inject(g, _field(g), 2, 1.0, 3, 7, 1, ppc, vth, (vd, 0.0, -0.3), 1.0)
    n = NC[1] * NC[2] * ppc
    assert len(inj["x"]) == n
    for comp, mu in (("u", vd), ("v", 0.0), ("w", -0.3)):
        a = inj[comp]
        assert abs(a.mean() - mu) < 5 * vth / math.sqrt(n)
        assert abs(a.std() - vth) < 5 * vth / math.sqrt(2 * n)
    # components uncorrelated
    assert abs(np.corrcoef(inj["u"], inj["v"])[0, 1]) < 5 / math.sqrt(n)


def test_determinism_and_cycle_dependence():
    g = O.make_grid(NC, LEN, bc=OPEN_X, dt=0.5)
    F = _field(g)
    a = O.inject(g, F, 0, 1.0, 3, 5, 2, 8, 0.1, (0.2, 0, 0), 1.0)
    b = O.inject(g, F, 0, 1.0, 3, 5, 2, 8, 0.1, (0.2, 0, 0), 1.0)
    c = O.inject(g, F, 0, 1.0, 3, 5, 3, 8, 0.1, (0.2, 0, 0), 1.0)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    assert not np.array_equal(a["x"][:10], c["x"][:10])
    assert not set(a["id"].tolist()) & set(c["id"].tolist())
