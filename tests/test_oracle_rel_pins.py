"""Pins of the relativistic oracle mover (NEXT-1: Eq. 2 with gamma, PAPER.md:149-165,
readings R4/R5/R6 of DESIGN.md §3), no GPU.

Expected values come from closed forms of the relativistic equations, not from
the oracle: the pure-B rotation angle 2 atan(|Omega| dt / (2 gamma)) with gamma,
|v| and v_par conserved (R4's derived guiding-centre factor; the printed 1/gamma
factor would make v_par grow), the orbit radius gamma v_perp / |Omega|, the exact
momentum kick u^{n+1} = u^n + (q/m) E dt in a uniform E, and the gamma -> 1 limit.
"""
import math

import numpy as np

import oracle as O
from test_oracle_pins import LEN, NC, const_field, parts1, pos, rodrigues, vel, window


def gamma(v, c):
    return 1.0 / math.sqrt(1.0 - np.dot(v, v) / (c * c))


def test_rel_gyration_angle_radius_guiding_centre():
    dt, qom, c = 0.5, 1.0, 1.0
    B = np.array([0.2, -0.1, 0.9])
    g = O.make_grid(NC, LEN, dt=dt, c=c)
    F = window(NC, 2, const_field((0, 0, 0), B), LEN)
    Om = qom * B / c
    v0 = np.array([0.5, 0.2, 0.3])           # |v| = 0.62 c, gamma = 1.27
    gm = gamma(v0, c)
    th = 2 * math.atan(np.linalg.norm(Om) * dt / (2 * gm))
    R = rodrigues(Om, -th)
    x0 = np.array([2.0, 2.0, 2.0])
    p = parts1(x0, v0)
    b = Om / np.linalg.norm(Om)
    vpar = v0.dot(b)
    vperp = np.linalg.norm(v0 - vpar * b)
    gc0 = x0 + gm * np.cross(v0, Om) / Om.dot(Om)
    v = v0.copy()
    for n in range(1, 16):
        st, bad = O.mover(g, F, qom, 3, p, relativistic=True)
        assert bad == 0 and st[0] == O.ALIVE
        v = R @ v
        np.testing.assert_allclose(vel(p), v, rtol=0, atol=1e-14)
        assert abs(np.linalg.norm(vel(p)) - np.linalg.norm(v0)) < 1e-14      # gamma conserved
        assert abs(vel(p).dot(b) - vpar) < 1e-14                              # R4 (derived form)
        x = pos(p)
        gc = x + gm * np.cross(vel(p), Om) / Om.dot(Om)
        d = gc - (gc0 + n * dt * vpar * b)
        d -= np.array(LEN) * np.round(d / np.array(LEN))      # periodic box: min image
        np.testing.assert_allclose(d, 0.0, rtol=0, atol=1e-13)
        r = np.linalg.norm(np.cross(x - gc, b))
        assert abs(r - gm * vperp / np.linalg.norm(Om)) < 1e-13


def test_rel_uniform_e_momentum_kick_and_position():
    """B = 0: u^{n+1} = u^n + (q/m) E dt exactly (any gamma-tilde), and with
    n_iter >= 2 gamma-tilde = (gamma^n + gamma^{n+1}) / 2, so
    x^{n+1} = x^n + dt (u^n + (q/m) E dt / 2) / gamma-tilde."""
    dt, qom, c = 0.25, -2.0, 1.0
    E = np.array([0.3, -0.4, 0.1])
    g = O.make_grid(NC, LEN, dt=dt, c=c)
    F = window(NC, 2, const_field(E, (0, 0, 0)), LEN)
    x = np.array([1.5, 2.0, 2.5])
    v = np.array([0.3, 0.1, -0.2])
    p = parts1(x, v)
    for n in range(6):
        gn = gamma(v, c)
        u = gn * v
        u1 = u + qom * E * dt
        g1 = math.sqrt(1.0 + u1.dot(u1) / (c * c))
        x = x + dt * (u + qom * E * dt / 2) / ((gn + g1) / 2)
        v = u1 / g1
        O.mover(g, F, qom, 3, p, relativistic=True)
        np.testing.assert_allclose(vel(p), v, rtol=1e-14, atol=1e-16)
        np.testing.assert_allclose(pos(p), x, rtol=1e-14, atol=1e-15)
        assert np.linalg.norm(vel(p)) < c


def test_rel_nonrelativistic_limit():
    """c -> large: the relativistic mover reduces to the gamma == 1 mover (R3)."""
    rng = np.random.default_rng(7)
    c = 1e7
    g = O.make_grid(NC, LEN, dt=0.5, c=c)
    nodes = rng.uniform(-1, 1, (NC[2] + 5, NC[1] + 5, NC[0] + 5, 6)) * np.array([1e-3] * 3 + [0.02 * c] * 3)
    F = O.FieldWindow((-2, -2, -2), nodes)
    n = 64
    base = {k: rng.uniform(1.0, 3.0, n) for k in "xyz"}
    base.update({k: rng.normal(0, 0.05, n) for k in "uvw"})
    base["q"] = np.ones(n)
    a = {k: v.copy() for k, v in base.items()}
    b = {k: v.copy() for k, v in base.items()}
    O.mover(g, F, -3.0, 3, a, relativistic=False)
    O.mover(g, F, -3.0, 3, b, relativistic=True)
    for k in "xyzuvw":
        np.testing.assert_allclose(b[k], a[k], rtol=1e-10, atol=1e-13)


def test_rel_superluminal_input_is_bad():
    """R23: |v| >= c has no gamma; the particle is flagged bad."""
    g = O.make_grid(NC, LEN, dt=0.5, c=1.0)
    F = window(NC, 2, const_field((0, 0, 0), (0, 0, 0.1)), LEN)
    p = parts1((2, 2, 2), (0.8, 0.7, 0.0))
    st, bad = O.mover(g, F, 1.0, 3, p, relativistic=True)
    assert bad == 1 and st[0] == O.BAD
