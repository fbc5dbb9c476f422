"""Pins of the CPU oracle against closed forms and brute force (no GPU).

Each test names the passage or reading it checks (SURVEY.md §8(c) P-numbers,
DESIGN.md §3 R-numbers).  None of the expected values below is produced by the
oracle itself: they come from closed-form solutions of Eq. 2 / Eq. 3, exact
rational arithmetic (``fractions``), numpy linear algebra (Rodrigues rotation),
or sums over the inputs.
"""
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


# ----------------------------------------------------------------- helpers --
def window(ncell, G, fn, length):
    """Field window over global nodes [-G, ncell+G] per axis, values fn(X,Y,Z)
    evaluated at node positions (analytic extension, no periodic mapping)."""
    n = [ncell[d] + 1 + 2 * G for d in range(3)]
    dl = [length[d] / ncell[d] for d in range(3)]
    xs = [(np.arange(n[d]) - G) * dl[d] for d in range(3)]
    Z, Y, X = np.meshgrid(xs[2], xs[1], xs[0], indexing="ij")
    EB = np.zeros((n[2], n[1], n[0], 6))
    vals = fn(X, Y, Z)
    for m in range(6):
        EB[..., m] = vals[m]
    return O.FieldWindow((-G, -G, -G), EB)


def periodic_window(ncell, G, node_vals):
    """Window replicating periodic images of node_vals[nz][ny][nx][6]."""
    idx = [np.arange(-G, ncell[d] + 1 + G) % ncell[d] for d in range(3)]
    EB = node_vals[np.ix_(idx[2], idx[1], idx[0])]
    return O.FieldWindow((-G, -G, -G), EB)


def const_field(E, B):
    def fn(X, Y, Z):
        one = np.ones_like(X)
        return [E[0] * one, E[1] * one, E[2] * one, B[0] * one, B[1] * one, B[2] * one]
    return fn


def parts1(x, v, q=1.0):
    return {"x": np.array([x[0]], float), "y": np.array([x[1]], float), "z": np.array([x[2]], float),
            "u": np.array([v[0]], float), "v": np.array([v[1]], float), "w": np.array([v[2]], float),
            "q": np.array([q], float)}


def pos(p, i=0):
    return np.array([p["x"][i], p["y"][i], p["z"][i]])


def vel(p, i=0):
    return np.array([p["u"][i], p["v"][i], p["w"][i]])


def rodrigues(axis, angle):
    k = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


NC, LEN = (16, 16, 16), (4.0, 4.0, 4.0)   # Delta = 0.25


# -------------------------------------------------------- field sampling ----
def test_sample_node_exact_and_cell_centre():
    """a node returns the node value; a cell centre the mean."""
    rng = np.random.default_rng(0)
    vals = rng.standard_normal((16, 16, 16, 6))
    g = O.make_grid(NC, LEN)
    F = periodic_window(NC, 2, vals)
    assert np.array_equal(O.sample(g, F, [5 * 0.25, 7 * 0.25, 3 * 0.25]), vals[3, 7, 5])
    got = O.sample(g, F, [5.5 * 0.25, 7.5 * 0.25, 3.5 * 0.25])
    want = vals[3:5, 7:9, 5:7].reshape(8, 6).mean(axis=0)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)


def test_sample_linear_reproduction():
    """trilinear interpolation reproduces linear fields."""
    g = O.make_grid(NC, LEN)
    F = window(NC, 2, lambda X, Y, Z: [X, Y, Z, 2 * X - Y + 0.5, 3 * Z + 1, X + Y + Z], LEN)
    rng = np.random.default_rng(1)
    for _ in range(200):
        p = rng.uniform(-0.2, 4.2, 3)
        got = O.sample(g, F, p)
        want = [p[0], p[1], p[2], 2 * p[0] - p[1] + 0.5, 3 * p[2] + 1, p.sum()]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-13)


def test_sample_bilinear_cross_term():
    """Trilinear is exact for xyz products inside a cell (catches a swapped f / 1-f)."""
    g = O.make_grid(NC, LEN)
    F = window(NC, 1, lambda X, Y, Z: [X * Y * Z, X * Y, Y * Z, X * Z, X * X * 0, X], LEN)
    p = np.array([1.3, 2.1, 0.7])
    # within one cell a trilinear interpolant of xyz equals the exact xyz only
    # at nodes; compare against the explicit 8-node formula instead:
    d = 0.25
    i = np.floor(p / d)
    f = p / d - i
    lo = i * d
    hi = lo + d
    def tri(fun):
        tot = 0.0
        for c in range(8):
            b = [(c >> k) & 1 for k in range(3)]
            w = np.prod([f[k] if b[k] else 1 - f[k] for k in range(3)])
            node = [hi[k] if b[k] else lo[k] for k in range(3)]
            tot += w * fun(*node)
        return tot
    got = O.sample(g, F, p)
    np.testing.assert_allclose(got[0], tri(lambda x, y, z: x * y * z), atol=1e-15)
    np.testing.assert_allclose(got[1], tri(lambda x, y, z: x * y), atol=1e-15)
    np.testing.assert_allclose(got[2], tri(lambda x, y, z: y * z), atol=1e-15)


# ------------------------------------------------------------------ mover ---
def test_p1_free_streaming():
    """P1: E = B = 0 -> v unchanged bit-exactly, x advances by v dt with wrap (R10)."""
    g = O.make_grid(NC, LEN, dt=0.5)
    F = window(NC, 2, const_field((0, 0, 0), (0, 0, 0)), LEN)
    p = parts1((3.9, 0.1, 2.0), (0.375, -0.5, 0.0625))
    v0 = vel(p).copy()
    for n in range(1, 9):
        O.mover(g, F, -256.0, 3, p)
        assert np.array_equal(vel(p), v0)
    want = np.mod(np.array([3.9, 0.1, 2.0]) + 8 * 0.5 * v0, 4.0)
    np.testing.assert_allclose(pos(p), want, rtol=0, atol=8 * 4.0 * 2.2e-16 * 4)


def test_wrap_examples():
    """SPEC.md:150-152 and R10: x = L + 0.1 dx wraps to 0.1 dx; inside is unchanged."""
    g = O.make_grid(NC, LEN, dt=1.0)
    F = window(NC, 2, const_field((0, 0, 0), (0, 0, 0)), LEN)
    p = parts1((3.95, 1.0, 1.0), (0.075, 0.0, 0.0))     # 3.95 + 0.075 = 4.025 = L + 0.1*dx
    O.mover(g, F, 1.0, 3, p)
    assert abs(p["x"][0] - 0.025) < 1e-15
    p = parts1((0.01, 1.0, 1.0), (-0.02, 0.0, 0.0))
    O.mover(g, F, 1.0, 3, p)
    assert abs(p["x"][0] - 3.99) < 1e-15
    p = parts1((2.0, 1.0, 1.0), (0.25, 0.0, 0.0))
    O.mover(g, F, 1.0, 3, p)
    assert p["x"][0] == 2.25


def test_p2_gyration_angle_radius_guiding_centre():
    """P2: uniform B, E = 0.  Per step v rotates about B by -2 atan(|Omega| dt/2)
    (q > 0), |v| is conserved, the guiding centre x + v x Omega/|Omega|^2 moves by
    v_par dt, and the orbit radius equals v_perp/|Omega| (Eq. 2 with gamma = 1)."""
    dt, qom, c = 0.5, 1.0, 1.0
    B = np.array([0.3, -0.2, 1.1])
    g = O.make_grid(NC, LEN, dt=dt, c=c)
    F = window(NC, 2, const_field((0, 0, 0), B), LEN)
    Om = qom * B / c
    th = 2 * math.atan(np.linalg.norm(Om) * dt / 2)
    R = rodrigues(Om, -th)
    x0 = np.array([2.0, 2.0, 2.0])
    v0 = np.array([0.01, 0.02, -0.005])
    p = parts1(x0, v0)
    gc0 = x0 + np.cross(v0, Om) / Om.dot(Om)
    vpar = v0.dot(Om) / np.linalg.norm(Om)
    vperp = np.linalg.norm(v0 - vpar * Om / np.linalg.norm(Om))
    v = v0.copy()
    for n in range(1, 21):
        O.mover(g, F, qom, 3, p)
        v = R @ v
        np.testing.assert_allclose(vel(p), v, rtol=0, atol=1e-16)
        assert abs(np.linalg.norm(vel(p)) - np.linalg.norm(v0)) < 1e-16
        x = pos(p)
        gc = x + np.cross(vel(p), Om) / Om.dot(Om)
        np.testing.assert_allclose(gc, gc0 + n * dt * vpar * Om / np.linalg.norm(Om), rtol=0, atol=1e-14)
        r = np.linalg.norm(np.cross(x - gc, Om / np.linalg.norm(Om)))
        assert abs(r - vperp / np.linalg.norm(Om)) < 1e-14


def test_p2_rotation_sign_electron():
    """P2/R8: the sense of rotation flips with the sign of q/m."""
    dt = 0.5
    g = O.make_grid(NC, LEN, dt=dt)
    F = window(NC, 2, const_field((0, 0, 0), (0, 0, 0.5)), LEN)
    for qom in (+1.0, -4.0):
        p = parts1((2, 2, 2), (0.01, 0, 0))
        O.mover(g, F, qom, 3, p)
        th = 2 * math.atan(abs(qom) * 0.5 * dt / 2)
        want = rodrigues((0, 0, 1), -math.copysign(th, qom)) @ np.array([0.01, 0, 0])
        np.testing.assert_allclose(vel(p), want, atol=1e-17)


def test_p3_exb_drift():
    """P3: starting at v_E = c E x B/|B|^2, E perpendicular to B, the particle drifts
    with v_E exactly; a general start rotates about v_E."""
    dt, c = 0.5, 1.0
    E = np.array([0.0, 1e-4, 0.0])
    B = np.array([0.0, 0.0, 0.01])
    vE = c * np.cross(E, B) / B.dot(B)
    g = O.make_grid(NC, LEN, dt=dt, c=c)
    F = window(NC, 2, const_field(E, B), LEN)
    for qom in (1.0, -256.0):
        p = parts1((1.0, 1.0, 1.0), vE)
        for n in range(1, 6):
            O.mover(g, F, qom, 3, p)
            np.testing.assert_allclose(vel(p), vE, rtol=0, atol=1e-17)
            np.testing.assert_allclose(pos(p), np.array([1.0, 1, 1]) + n * dt * vE, rtol=0, atol=1e-15)
    qom = 1.0
    Om = qom * B / c
    th = 2 * math.atan(np.linalg.norm(Om) * dt / 2)
    R = rodrigues(Om, -th)
    v0 = np.array([0.003, -0.002, 0.0])
    p = parts1((1.0, 1.0, 1.0), v0)
    for n in range(1, 6):
        O.mover(g, F, qom, 3, p)
        want = vE + np.linalg.matrix_power(R, n) @ (v0 - vE)
        np.testing.assert_allclose(vel(p), want, rtol=0, atol=1e-17)


def test_p4_uniform_e_bit_exact():
    """P4 / SPEC.md:142 / R7: B = 0, uniform E: v^n = v^0 + n (q/m) E dt,
    x^n = x^0 + n v^0 dt + n^2 (q/m) E dt^2 / 2, bit-exact on dyadic inputs."""
    g = O.make_grid(NC, LEN, dt=0.125)
    F = window(NC, 2, const_field((1.0, -0.5, 0.25), (0, 0, 0)), LEN)
    qom = 0.5
    p = parts1((1.0, 2.0, 3.0), (0.0, 0.125, 0.0))
    x0, v0, E = np.array([1.0, 2.0, 3.0]), np.array([0.0, 0.125, 0.0]), np.array([1.0, -0.5, 0.25])
    for n in range(1, 5):
        O.mover(g, F, qom, 3, p)
        assert np.array_equal(vel(p), v0 + n * qom * E * 0.125)
        assert np.array_equal(pos(p), x0 + n * v0 * 0.125 + n * n * qom * E * 0.125 ** 2 / 2)
    # SPEC.md:142 worked example: v = 0, E = (1,0,0), q/m = 1, dt = 0.1 -> v = (0.1, 0, 0)
    g = O.make_grid(NC, LEN, dt=0.1)
    F = window(NC, 2, const_field((1.0, 0, 0), (0, 0, 0)), LEN)
    p = parts1((1.0, 1.0, 1.0), (0, 0, 0))
    O.mover(g, F, 1.0, 3, p)
    np.testing.assert_allclose(vel(p), [0.1, 0, 0], rtol=1e-15)


def test_p5_e_parallel_b():
    """P5: E parallel to B: the parallel velocity gains (q/m) E dt per step and the
    perpendicular velocity rotates as in P2 (superposition)."""
    dt, qom = 0.25, -2.0
    b = np.array([1.0, 2.0, 2.0]) / 3.0
    E, B = 1e-3 * b, 0.4 * b
    g = O.make_grid(NC, LEN, dt=dt)
    F = window(NC, 2, const_field(E, B), LEN)
    Om = qom * B
    R = rodrigues(Om, -2 * math.atan(np.linalg.norm(Om) * dt / 2))
    v0 = np.array([0.01, -0.02, 0.005])
    vpar0 = v0.dot(b)
    vperp = v0 - vpar0 * b
    p = parts1((2, 2, 2), v0)
    for n in range(1, 8):
        O.mover(g, F, qom, 3, p)
        vperp = R @ vperp
        want = vperp + (vpar0 + n * qom * 1e-3 * dt) * b
        np.testing.assert_allclose(vel(p), want, rtol=0, atol=1e-16)


def _golden_p6():
    rows = {}
    with open(os.path.join(HERE, "golden", "p6_linear_field.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, xs, vs = line.split()
            rows[int(k)] = (Fr(xs), Fr(vs))
    return rows


def test_p6_linear_field_worked_example():
    """P6 (R1, R2): the golden values equal the affine recursion of Eq. 2 solved in
    exact rationals, and the fp64 oracle reproduces them bit-for-bit."""
    gold = _golden_p6()
    alpha, k, dt, xn, vn = Fr(1, 2), Fr(1, 4), Fr(1, 2), Fr(1), Fr(1, 4)
    for n_iter, (xg, vg) in gold.items():
        vb = vn + k * alpha * xn                       # R1: first sample at x^n
        for _ in range(n_iter - 1):
            vb = vn + k * alpha * (xn + vb * dt / 2)
        assert (xn + vb * dt, 2 * vb - vn) == (xg, vg)
        g = O.make_grid(NC, LEN, dt=0.5)
        F = window(NC, 2, lambda X, Y, Z: [0.5 * X, 0 * X, 0 * X, 0 * X, 0 * X, 0 * X], LEN)
        p = parts1((1.0, 1.0, 1.0), (0.25, 0.0, 0.0))
        O.mover(g, F, 1.0, n_iter, p)
        assert p["x"][0] == float(xg) and p["u"][0] == float(vg)


def test_open_boundary_removal_and_planet():
    """R21: leaving through an open face or entering the planet removes."""
    g = O.make_grid(NC, LEN, bc=(O.OPEN, O.OPEN, O.PERIODIC), dt=1.0,
                    planet_center=(2.0, 2.0, 2.0), planet_radius=0.5)
    F = window(NC, 2, const_field((0, 0, 0), (0, 0, 0)), LEN)
    p = {k: np.array(v, float) for k, v in dict(
        x=[3.9, 0.05, 1.0, 1.2, 2.0], y=[1.0, 1.0, 3.99, 2.0, 1.0], z=[1, 1, 1, 2.0, 3.95],
        u=[0.2, -0.1, 0.0, 0.5, 0.0], v=[0.0, 0.0, 0.02, 0.0, 0.0], w=[0.0, 0.0, 0.0, 0.0, 0.1]).items()}
    st, bad = O.mover(g, F, 1.0, 3, p)
    assert list(st) == [O.REMOVED, O.REMOVED, O.REMOVED, O.REMOVED, O.ALIVE]
    assert abs(p["z"][4] - 0.05) < 1e-15          # periodic axis still wraps


def test_fixed_count_no_early_exit():
    """R2: n_iter = 1, 2, 3 give different results (no convergence test)."""
    g = O.make_grid(NC, LEN, dt=0.5)
    F = window(NC, 2, lambda X, Y, Z: [0.5 * X, 0 * X, 0 * X, 0 * X, 0 * X, 0.2 + 0 * X], LEN)
    res = []
    for n_iter in (1, 2, 3, 4):
        p = parts1((1.0, 1.0, 1.0), (0.25, 0.1, 0.0))
        O.mover(g, F, 1.0, n_iter, p)
        res.append((p["x"][0], p["u"][0]))
    assert len(set(res)) == 4


# ---------------------------------------------------------------- moments ---
def test_p7_single_particle_node_and_centre():
    """P7 / SPEC.md:205-206, 214: q/V at the node; q/(8V) at 8 nodes from a cell
    centre; v = (1,0,0) gives J_x = Pi_xx = rho."""
    g = O.make_grid(NC, LEN)
    V = 0.25 ** 3
    mom, _ = O.moments(g, parts1((5 * 0.25, 6 * 0.25, 7 * 0.25), (1.0, 0, 0), q=3.0))
    assert mom[0, 7, 6, 5] == 3.0 / V
    assert np.count_nonzero(mom[0]) == 1
    assert mom[1, 7, 6, 5] == 3.0 / V and mom[4, 7, 6, 5] == 3.0 / V
    assert np.count_nonzero(mom[[2, 3, 5, 6, 7, 8, 9]]) == 0
    mom, _ = O.moments(g, parts1((5.5 * 0.25, 6.5 * 0.25, 7.5 * 0.25), (0, 0, 0), q=2.0))
    assert np.count_nonzero(mom[0]) == 8
    assert np.all(mom[0, 7:9, 6:8, 5:7] == 2.0 / (8 * V))


def test_p7_periodic_fold():
    """R18: a particle in the last cell deposits on node N == node 0."""
    g = O.make_grid(NC, LEN)
    V = 0.25 ** 3
    mom, _ = O.moments(g, parts1((15.5 * 0.25, 0.0, 0.0), (0, 0, 0), q=1.0))
    assert mom[0, 0, 0, 15] == 0.5 / V and mom[0, 0, 0, 0] == 0.5 / V


def _random_parts(rng, n, length, vth=0.1, qrange=(0.5, 1.5)):
    return {"x": rng.uniform(0, length[0], n), "y": rng.uniform(0, length[1], n),
            "z": rng.uniform(0, length[2], n), "u": rng.normal(0, vth, n),
            "v": rng.normal(0, vth, n), "w": rng.normal(0, vth, n), "q": rng.uniform(*qrange, n)}


@pytest.mark.parametrize("bc", [(0, 0, 0), (1, 1, 1), (1, 0, 1)])
def test_p8_global_sums(bc):
    """P8 (R13, R14, R18): sum_g rho V = sum q; sum_g J V = sum q v; sum_g Pi V = sum q v v."""
    rng = np.random.default_rng(7)
    g = O.make_grid((8, 6, 5), (2.0, 1.5, 1.25), bc=bc)
    p = _random_parts(rng, 5000, (2.0, 1.5, 1.25))
    V = 0.25 ** 3
    mom, am = O.moments(g, p)
    q, v = p["q"], np.stack([p["u"], p["v"], p["w"]])
    want = [q.sum()] + [(q * v[a]).sum() for a in range(3)] + \
           [(q * v[a] * v[b]).sum() for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))]
    absw = [np.abs(q).sum()] + [np.abs(q * v[a]).sum() for a in range(3)] + \
           [np.abs(q * v[a] * v[b]).sum() for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))]
    for m in range(10):
        assert abs(mom[m].sum() * V - want[m]) <= 1e-13 * absw[m]
        assert abs(am[m].sum() * V - absw[m]) <= 1e-13 * absw[m]


def test_p9_adjointness():
    """P9 / SPEC.md:237: sum_g phi_g rho_g V = sum_p q_p phi(x_p) with the gather W."""
    rng = np.random.default_rng(3)
    nc, ln = (8, 6, 5), (2.0, 1.5, 1.25)
    g = O.make_grid(nc, ln)
    p = _random_parts(rng, 400, ln)
    phi = rng.standard_normal((nc[2], nc[1], nc[0]))
    vals = np.zeros((nc[2], nc[1], nc[0], 6))
    vals[..., 0] = phi
    F = periodic_window(nc, 1, vals)
    gathered = sum(p["q"][i] * O.sample(g, F, [p["x"][i], p["y"][i], p["z"][i]])[0]
                   for i in range(400))
    mom, _ = O.moments(g, p)
    assert abs((phi * mom[0]).sum() * 0.25 ** 3 - gathered) < 1e-12 * np.abs(p["q"]).sum() * np.abs(phi).max()


def test_p10_lattice_loading():
    """P10: 27 particles per cell on the sub-lattice ((k+1/2)/3) Delta give uniform rho."""
    nc = (4, 4, 4)
    g = O.make_grid(nc, (1.0, 1.0, 1.0))
    d = 0.25
    sub = (np.arange(3) + 0.5) / 3
    cells = np.arange(4)
    xs = ((cells[:, None] + sub[None, :]) * d).ravel()
    Z, Y, X = np.meshgrid(xs, xs, xs, indexing="ij")
    n = X.size
    p = {"x": X.ravel().copy(), "y": Y.ravel().copy(), "z": Z.ravel().copy(),
         "u": np.zeros(n), "v": np.zeros(n), "w": np.zeros(n), "q": np.full(n, 0.5)}
    mom, _ = O.moments(g, p)
    np.testing.assert_allclose(mom[0], 27 * 0.5 / d ** 3, rtol=1e-14)


def test_p11_dyadic_brute_force():
    """P11 (R19): dyadic inputs -> every product and sum is exact, so the oracle must
    equal an exact-rational brute-force deposit of Eq. 3 bit-for-bit."""
    rng = np.random.default_rng(11)
    nc, ln = (4, 4, 4), (1.0, 1.0, 1.0)
    g = O.make_grid(nc, ln)
    for trial in range(20):
        n = int(rng.integers(1, 9))
        P = {k: (rng.integers(0, 64, n) / 64.0) for k in "xyz"}
        for k in "uvw":
            P[k] = rng.integers(-8, 9, n) / 8.0
        P["q"] = rng.integers(1, 5, n) / 4.0
        mom, _ = O.moments(g, P)
        exact = np.zeros_like(mom, dtype=object)
        exact[...] = Fr(0)
        V = Fr(1, 64)
        for i in range(n):
            xi = [Fr(P[k][i]) / Fr(1, 4) for k in "xyz"]
            cell = [math.floor(t) for t in xi]
            f = [xi[d] - cell[d] for d in range(3)]
            v = [Fr(P[k][i]) for k in "uvw"]
            q = Fr(P["q"][i])
            vals = [1, v[0], v[1], v[2], v[0] * v[0], v[0] * v[1], v[0] * v[2], v[1] * v[1], v[1] * v[2], v[2] * v[2]]
            for c in range(8):
                b = [(c >> k) & 1 for k in range(3)]
                S = Fr(1)
                for d in range(3):
                    S *= f[d] if b[d] else 1 - f[d]
                node = [(cell[d] + b[d]) % 4 for d in range(3)]
                for m in range(10):
                    exact[m, node[2], node[1], node[0]] += q * vals[m] * S / V
        assert np.array_equal(mom, exact.astype(float)), trial


def test_p12_pressure_trace_and_sign():
    """P12 (R16): tr Pi = rho of the same particles with charge q |v|^2; Pi_xx >= 0 for q > 0."""
    rng = np.random.default_rng(5)
    g = O.make_grid((8, 6, 5), (2.0, 1.5, 1.25))
    p = _random_parts(rng, 2000, (2.0, 1.5, 1.25))
    mom, am = O.moments(g, p)
    p2 = dict(p)
    p2["q"] = p["q"] * (p["u"] ** 2 + p["v"] ** 2 + p["w"] ** 2)
    mom2, _ = O.moments(g, p2)
    np.testing.assert_allclose(mom[4] + mom[7] + mom[9], mom2[0], rtol=1e-13, atol=1e-13 * mom2[0].max())
    assert np.all(mom[4] >= 0) and np.all(mom[7] >= 0) and np.all(mom[9] >= 0)


def test_removed_particles_excluded():
    """R15: removed particles do not deposit."""
    g = O.make_grid((4, 4, 4), (1.0, 1.0, 1.0), bc=(1, 1, 1))
    p = parts1((0.3, 0.3, 0.3), (0, 0, 0))
    st = np.array([O.REMOVED], dtype=np.int8)
    mom, _ = O.moments(g, p, status=st)
    assert not mom.any()


# ------------------------------------------ R11: the clamp to the window ----
def test_sample_clamp_branch_linear_field_closed_form():
    """R11: a position outside the field window is clamped to
    the window box (constant extension along the outward normal).  For a linear
    field the trilinear sample at the clamped point is the field there, so the
    expected value is the linear function evaluated at clip(p, box) -- a closed
    form that does not use the oracle.  Positions beyond every face, edge and
    corner of the box, and NaN (clamped to the low face), are covered; the
    clamp flag is set exactly when a coordinate is outside."""
    G = 2
    g = O.make_grid(NC, LEN, bc=(O.OPEN,) * 3)
    fn = lambda X, Y, Z: [X, 2 * Y - 1, 0.5 * Z + X, -Y + 3, Z - X, 0.25 * X + Y + Z]
    F = window(NC, G, fn, LEN)
    d = LEN[0] / NC[0]
    lo, hi = -G * d, (NC[0] + G) * d          # window box per axis (cubic here)
    rng = np.random.default_rng(11)
    checked = 0
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            for sz in (-1, 0, 1):
                for _ in range(6):
                    p = rng.uniform(lo + 0.01, hi - 0.01, 3)
                    for ax, sgn in enumerate((sx, sy, sz)):
                        if sgn < 0:
                            p[ax] = lo - rng.uniform(1e-9, 5.0)
                        elif sgn > 0:
                            p[ax] = hi + rng.uniform(1e-9, 5.0)
                    c = np.clip(p, lo, hi)
                    got, flag = O.sample_ex(g, F, p)
                    np.testing.assert_allclose(got, fn(*c), rtol=0, atol=1e-12)
                    assert flag == int((sx, sy, sz) != (0, 0, 0))
                    checked += 1
    assert checked == 27 * 6
    # exactly on the top face: inside (no clamp), value of the face
    p = np.array([hi, 1.0, 1.0])
    got, flag = O.sample_ex(g, F, p)
    assert flag == 0
    np.testing.assert_allclose(got, fn(*p), rtol=0, atol=1e-12)
    # NaN coordinate: clamped to the low face, flagged
    got, flag = O.sample_ex(g, F, np.array([np.nan, 1.0, 1.0]))
    assert flag == 1
    np.testing.assert_allclose(got, fn(lo, 1.0, 1.0), rtol=0, atol=1e-12)
