"""Pins of the NEXT-2 oracle: susceptibility chi (Eq. 5) and corrected sources
rho-hat, J-hat (Eq. 6), readings R24-R27 of DESIGN.md §3.

Expected values are not produced by oracle_implicit_sources itself: the B = 0
and rho = 0 limits, the exact linear response of the oracle MOVER (push_one,
a separate code path) to a small E in uniform B — which is what R_s must be for
Eq. 4 to embed Eq. 2 — and the closed form of the discrete central difference of
a single Fourier mode, sin(k(x+d)) - sin(k(x-d)) = 2 cos(kx) sin(kd).
"""
import math

import numpy as np

import oracle as O
from test_oracle_pins import const_field, parts1, vel, window

FOUR_PI = 4.0 * math.pi


def grid(n=(8, 6, 4), L=(2.0, 1.5, 1.0), bc=(0, 0, 0), dt=0.3, c=1.0):
    return O.make_grid(n, L, bc=bc, dt=dt, c=c)


def nodes(g):
    nx, ny, nz = O.node_counts(g)
    return nx, ny, nz


def test_chi_b_zero_is_isotropic():
    g = grid()
    nx, ny, nz = nodes(g)
    rng = np.random.default_rng(1)
    qoms = [-256.0, 1.0]
    moms = []
    for qom in qoms:
        m = np.zeros((10, nz, ny, nx))
        m[0] = np.sign(qom) * rng.uniform(0.1, 1.0, (nz, ny, nx))   # rho_s has the sign of q_s
        moms.append(m)
    chi, _, _ = O.implicit_sources(g, qoms, moms, np.zeros((nz, ny, nx, 3)))
    w2dt2 = sum(FOUR_PI * m[0] * q for m, q in zip(moms, qoms)) * g.dt * g.dt
    assert (w2dt2 > 0).all()                                          # R24
    for r in range(3):
        for c in range(3):
            want = 0.5 * w2dt2 if r == c else 0.0
            np.testing.assert_allclose(chi[3 * r + c], want, rtol=1e-14, atol=0)


def test_chi_rho_zero_is_zero():
    g = grid()
    nx, ny, nz = nodes(g)
    B = np.random.default_rng(2).normal(size=(nz, ny, nx, 3))
    chi, _, _ = O.implicit_sources(g, [1.0], [np.zeros((10, nz, ny, nx))], B)
    assert not chi.any()


def test_chi_is_the_movers_linear_response():
    """R_s (Eq. 5, with R25's normalisation) equals the mover's response: a
    particle at rest in uniform B and a small uniform E gets, after one
    iterate of Eq. 2, v^{n+1} = 2 vb = 2 R (qom dt/2) E."""
    dt, c = 0.4, 1.0
    B = np.array([0.7, -0.3, 1.2])
    for qom in (1.0, -3.0):
        g = grid(dt=dt, c=c)
        nx, ny, nz = nodes(g)
        m = np.zeros((10, nz, ny, nx))
        m[0] = np.sign(qom) * 0.5
        Bn = np.broadcast_to(B, (nz, ny, nx, 3)).copy()
        chi, _, _ = O.implicit_sources(g, [qom], [m], Bn)
        chi_node = chi[:, 1, 2, 3].reshape(3, 3)
        scale = 0.5 * FOUR_PI * 0.5 * abs(qom) * dt * dt
        for E in (np.array([1e-3, 0, 0]), np.array([0, 2e-3, 0]), np.array([0.5e-3, -1e-3, 3e-3])):
            gm = O.make_grid((16, 16, 16), (4.0, 4.0, 4.0), dt=dt, c=c)
            F = window((16, 16, 16), 2, const_field(E, B), (4.0, 4.0, 4.0))
            p = parts1((2.0, 2.0, 2.0), (0.0, 0.0, 0.0))
            O.mover(gm, F, qom, 1, p)
            response = vel(p) / (2.0 * qom * dt / 2.0)                  # = R E
            np.testing.assert_allclose(chi_node @ E / scale, response, rtol=1e-12, atol=1e-18)


def _mode(g, axis, k):
    nx, ny, nz = nodes(g)
    d = g.len[axis] / g.ncell[axis]
    idx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    pos = idx[2 - axis] * d
    return np.sin(k * pos), np.cos(k * pos), d


def test_hat_b_zero_pi_zero_single_mode():
    """B = 0, Pi = 0: J-hat = J and rho-hat = rho - dt div J; for J_x = sin(kx)
    the discrete divergence is exactly cos(kx) sin(k dx) / dx."""
    g = grid(n=(16, 4, 4), L=(2.0, 1.0, 1.0))
    nx, ny, nz = nodes(g)
    k = 2 * math.pi / g.len[0] * 3
    s, c, d = _mode(g, 0, k)
    m = np.zeros((10, nz, ny, nx))
    m[0] = 0.7
    m[1] = s
    _, rh, jh = O.implicit_sources(g, [1.0], [m], np.zeros((nz, ny, nx, 3)))
    np.testing.assert_allclose(jh[0], s, rtol=0, atol=1e-15)
    assert not jh[1].any() and not jh[2].any()
    np.testing.assert_allclose(rh, 0.7 - g.dt * c * math.sin(k * d) / d, rtol=0, atol=1e-13)


def test_hat_uniform_j_keeps_rho():
    g = grid()
    nx, ny, nz = nodes(g)
    m = np.zeros((10, nz, ny, nx))
    m[0] = 0.3
    m[1:4] = np.array([0.1, -0.2, 0.05])[:, None, None, None]
    _, rh, _ = O.implicit_sources(g, [1.0], [m], np.zeros((nz, ny, nx, 3)))
    np.testing.assert_allclose(rh, 0.3, rtol=1e-15, atol=0)


def test_hat_pressure_divergence_single_mode():
    """B = 0: J-hat_y = J_y - (dt/2) d Pi_yz / dz with Pi_yz = sin(kz)."""
    g = grid(n=(4, 4, 16), L=(1.0, 1.0, 2.0))
    nx, ny, nz = nodes(g)
    k = 2 * math.pi / g.len[2] * 2
    s, c, d = _mode(g, 2, k)
    m = np.zeros((10, nz, ny, nx))
    m[0] = 1.0
    m[8] = s                                   # Pi_yz
    _, _, jh = O.implicit_sources(g, [1.0], [m], np.zeros((nz, ny, nx, 3)))
    np.testing.assert_allclose(jh[1], -(g.dt / 2) * c * math.sin(k * d) / d, rtol=0, atol=1e-14)
    assert np.abs(jh[0]).max() < 1e-15


def test_hat_open_axis_linear_field_exact():
    """Open axis: interior central and boundary one-sided differences (R27) are
    both exact for a linear J_x = alpha x, so div J = alpha at every node."""
    g = grid(n=(8, 4, 4), L=(2.0, 1.0, 1.0), bc=(1, 0, 0))
    nx, ny, nz = nodes(g)
    assert nx == 9
    d = g.len[0] / g.ncell[0]
    x = np.arange(nx) * d
    m = np.zeros((10, nz, ny, nx))
    m[0] = 0.5
    m[1] = 0.8 * x[None, None, :]
    _, rh, _ = O.implicit_sources(g, [1.0], [m], np.zeros((nz, ny, nx, 3)))
    np.testing.assert_allclose(rh, 0.5 - g.dt * 0.8, rtol=0, atol=1e-14)


def test_chi_uniform_bz_closed_form():
    """B = (0, 0, Bz): R = [[1, a, 0], [-a, 1, 0], [0, 0, 1 + a^2]] / (1 + a^2)
    with a = qom Bz dt / (2c), from x - a x x + (a.x) a."""
    g = grid(dt=0.5)
    nx, ny, nz = nodes(g)
    qom, Bz = -2.0, 0.8
    m = np.zeros((10, nz, ny, nx))
    m[0] = -0.25
    Bn = np.zeros((nz, ny, nx, 3))
    Bn[..., 2] = Bz
    chi, _, _ = O.implicit_sources(g, [qom], [m], Bn)
    a = qom * Bz * g.dt / 2
    R = np.array([[1, a, 0], [-a, 1, 0], [0, 0, 1 + a * a]]) / (1 + a * a)
    scale = 0.5 * FOUR_PI * (-0.25) * qom * g.dt ** 2
    np.testing.assert_allclose(chi[:, 0, 0, 0].reshape(3, 3), scale * R, rtol=1e-14, atol=1e-16)
