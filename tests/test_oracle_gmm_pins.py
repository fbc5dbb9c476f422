"""Pins of the NEXT-4 oracle (velocity binning and the
Gaussian-mixture fit by EM; readings R32-R33 of DESIGN.md §3), no GPU.

Expected values come from the inputs and closed forms, not from the oracle:
single-particle and mirrored bins, histogram moments against sample moments
within the bin-width (Sheppard) bound, one EM iteration with M = 1 equals the
histogram's weighted mean and covariance (+ eps), a single occupied bin, and a
two-component mixture recovered from samples.
"""
import math

import numpy as np

import oracle as O


def parts_from(vel, q=None):
    n = len(vel)
    return {"u": np.ascontiguousarray(vel[:, 0]), "v": np.ascontiguousarray(vel[:, 1]),
            "w": np.ascontiguousarray(vel[:, 2]), "q": np.ones(n) if q is None else q}


def centres(B, vmax):
    bw = 2 * vmax / B
    c = -vmax + (np.arange(B) + 0.5) * bw
    Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
    return np.stack([X, Y, Z], -1)


def test_single_particle_and_mirror_and_clip():
    B, vmax = 8, 1.0
    h, c = O.bin_velocities(parts_from(np.array([[0.125, -0.375, 0.875]]), np.array([-2.5])), None, B, vmax)
    assert c == 0 and h.sum() == 2.5
    assert h[7, 2, 4] == 2.5          # bins floor((v + 1) / 2 * 8): x 4, y 2, z 7
    h, c = O.bin_velocities(parts_from(np.array([[0.3, -0.6, 0.1], [-0.3, 0.6, -0.1]])), None, B, vmax)
    nz = np.argwhere(h > 0)
    assert len(nz) == 2 and (nz[0] + nz[1] == B - 1).all()   # mirrored about the centre
    h, c = O.bin_velocities(parts_from(np.array([[3.0, 0.0, 0.0], [0.0, -7.0, 0.0]])), None, B, vmax)
    assert c == 2 and h[4, 4, 7] == 1 and h[4, 0, 4] == 1


def test_histogram_moments_match_sample():
    rng = np.random.default_rng(4)
    vel = rng.normal([0.1, -0.05, 0.0], [0.2, 0.1, 0.15], (400000, 3))
    B, vmax = 48, 1.5
    h, c = O.bin_velocities(parts_from(vel), None, B, vmax)
    assert c == 0
    C = centres(B, vmax).reshape(-1, 3)
    w = h.reshape(-1)
    mean = (w[:, None] * C).sum(0) / w.sum()
    var = (w[:, None] * (C - mean) ** 2).sum(0) / w.sum()
    bw = 2 * vmax / B
    assert np.all(np.abs(mean - vel.mean(0)) < bw / 2)
    # binned variance = sample variance + bw^2/12 (Sheppard) within statistical noise
    np.testing.assert_allclose(var, vel.var(0) + bw * bw / 12, rtol=0.02)


def test_em_single_component_is_weighted_moments():
    rng = np.random.default_rng(5)
    B, vmax = 16, 1.0
    h = rng.uniform(0, 1, (B, B, B)) * (rng.uniform(0, 1, (B, B, B)) < 0.3)
    a, mu, sg = O.fit_gmm(h, vmax, 1, 1)
    C = centres(B, vmax).reshape(-1, 3)
    w = h.reshape(-1)
    m = (w[:, None] * C).sum(0) / w.sum()
    cov = np.einsum("b,bi,bj->ij", w, C - m, C - m) / w.sum()
    eps = 1e-6 * (2 * vmax / B) ** 2
    assert a[0] == 1.0 or abs(a[0] - 1) < 1e-15
    np.testing.assert_allclose(mu[0], m, rtol=1e-12, atol=1e-15)
    want = [cov[0, 0] + eps, cov[0, 1], cov[0, 2], cov[1, 1] + eps, cov[1, 2], cov[2, 2] + eps]
    np.testing.assert_allclose(sg[0], want, rtol=1e-10, atol=1e-15)


def test_em_single_bin_degenerate():
    B, vmax = 8, 1.0
    h = np.zeros((B, B, B))
    h[3, 5, 2] = 4.0
    a, mu, sg = O.fit_gmm(h, vmax, 1, 3)
    bw = 2 * vmax / B
    np.testing.assert_allclose(mu[0], [-vmax + 2.5 * bw, -vmax + 5.5 * bw, -vmax + 3.5 * bw], atol=1e-15)
    eps = 1e-6 * bw * bw
    np.testing.assert_allclose(sg[0], [eps, 0, 0, eps, 0, eps], rtol=1e-9, atol=1e-20)


def test_em_two_separated_components():
    rng = np.random.default_rng(6)
    v1 = rng.normal([-0.4, 0.0, 0.1], 0.08, (150000, 3))
    v2 = rng.normal([0.35, 0.2, -0.1], 0.06, (150000, 3))
    B, vmax = 32, 1.0
    h, _ = O.bin_velocities(parts_from(np.vstack([v1, v2])), None, B, vmax)
    a, mu, sg = O.fit_gmm(h, vmax, 2, 60)
    order = np.argsort(mu[:, 0])
    a, mu = a[order], mu[order]
    np.testing.assert_allclose(a, [0.5, 0.5], atol=0.02)
    np.testing.assert_allclose(mu[0], [-0.4, 0.0, 0.1], atol=0.05)
    np.testing.assert_allclose(mu[1], [0.35, 0.2, -0.1], atol=0.05)
    # component spreads near the sampled sigma^2 (+ Sheppard's bw^2/12)
    bw = 2 * vmax / B
    sg = sg[order]
    assert abs(sg[0][0] - (0.08 ** 2 + bw * bw / 12)) < 0.002 and abs(sg[1][3] - (0.06 ** 2 + bw * bw / 12)) < 0.002
