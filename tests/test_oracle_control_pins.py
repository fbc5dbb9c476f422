"""Pins of the NEXT-3 particle-control oracle (readings
R29-R31 of DESIGN.md §3), no GPU: splitting and pair-wise coalescence.

Expected values are conservation laws and closed forms, not oracle output:
splitting conserves charge, momentum, q|v|^2 exactly and the charge centroid to
rounding, keeps children in the parent's cell and splits a binomial number of
particles; coalescence conserves charge, momentum and the charge centroid, loses
exactly sum q1 q2/(q1+q2) |v1-v2|^2 of sum q|v|^2, merges only particles of one
cell and one velocity bin, and reproduces a hand-worked four-particle case.
"""
import math

import numpy as np

import oracle as O

NC, LEN = (8, 8, 8), (2.0, 2.0, 2.0)        # Delta = 0.25


def plasma(n, seed=3, vth=0.1):
    rng = np.random.default_rng(seed)
    p = {k: rng.uniform(0.0, 2.0, n) for k in "xyz"}
    p.update({k: rng.normal(0, vth, n) for k in "uvw"})
    p["q"] = rng.uniform(0.5, 1.5, n) * 1e-3
    p["id"] = np.arange(n, dtype=np.int64) * 7 + 11
    return p


def sums(p, st):
    a = st == O.ALIVE
    q = p["q"][a]
    v = np.stack([p["u"][a], p["v"][a], p["w"][a]])
    x = np.stack([p["x"][a], p["y"][a], p["z"][a]])
    return q.sum(), (q * v).sum(1), (q * (v * v).sum(0)).sum(), (q * x).sum(1)


def test_split_conserves_and_stays_in_cell():
    g = O.make_grid(NC, LEN, bc=(1, 1, 1), dt=0.5)
    p = plasma(4000)
    st = np.zeros(4000, dtype=np.int8)
    Q0, P0, E0, X0 = sums(p, st)
    # with a tiny displacement no split is rejected: the count is Binomial(n, p)
    tiny, _ = O.split(g, 1, p, st, 0.3, 1e-9, 77, 5)
    assert abs(len(tiny["x"]) - 4000 - 0.3 * 4000) < 5 * math.sqrt(4000 * 0.3 * 0.7)
    out, st2 = O.split(g, 1, p, st, 0.3, 0.1, 77, 5)
    Q1, P1, E1, X1 = sums(out, st2)
    nsplit = len(out["x"]) - 4000
    assert 0 < nsplit <= len(tiny["x"]) - 4000      # splits leaving the cell are skipped
    assert Q1 == Q0 or abs(Q1 - Q0) < 1e-16 * abs(Q0) * 4000
    np.testing.assert_allclose(P1, P0, rtol=1e-13, atol=1e-18)
    assert abs(E1 - E0) < 1e-13 * E0
    np.testing.assert_allclose(X1, X0, rtol=1e-13)
    # children: same velocity and cell as the parent (parent = slot, child 2 = appended)
    ids = out["id"]
    assert len(np.unique(ids)) == len(ids)
    child = ids >= (1 << 61)
    assert child.sum() == nsplit
    pos = {int(i): k for k, i in enumerate(ids)}
    d = LEN[0] / NC[0]
    for k in np.nonzero(child)[0][:200]:
        par = [j for j in range(4000) if O.child_id(int(ids[j]), 5) == int(ids[k])]
        assert len(par) == 1
        j = par[0]
        assert out["u"][j] == out["u"][k] and out["q"][j] == out["q"][k] == p["q"][j] / 2
        for c in "xyz":
            assert math.floor(out[c][j] / d) == math.floor(out[c][k] / d) == math.floor(p[c][j] / d)
            # the two children straddle the parent's position symmetrically
            assert abs(0.5 * (out[c][j] + out[c][k]) - p[c][j]) < 1e-15
    assert pos  # ids indexable


def test_coalesce_conservation_and_energy_loss():
    g = O.make_grid(NC, LEN, bc=(1, 1, 1), dt=0.5)
    p = plasma(6000, seed=9, vth=0.05)
    st = np.zeros(6000, dtype=np.int8)
    before = {k: v.copy() for k, v in p.items()}
    Q0, P0, E0, X0 = sums(p, st)
    dv = 0.05
    m = O.coalesce(g, p, st, dv, 0.2)
    assert m > 0 and (st == O.MERGED).sum() == m
    Q1, P1, E1, X1 = sums(p, st)
    assert abs(Q1 - Q0) < 1e-15 * Q0
    np.testing.assert_allclose(P1, P0, rtol=1e-12, atol=1e-17)
    np.testing.assert_allclose(X1, X0, rtol=1e-13)
    # energy loss: each merge removes q1 q2/(q1+q2)|v1-v2|^2, computed from the
    # partners recovered by their ids (keeper = smaller id, in the same cell and bins)
    d = LEN[0] / NC[0]
    lost = 0.0
    keepers = np.nonzero((st == O.ALIVE) & (np.abs(p["q"] - before["q"]) > 0))[0]
    gone = np.nonzero(st == O.MERGED)[0]
    assert len(keepers) == m
    cell = lambda k: tuple(int(math.floor(before[c][k] / d)) for c in "xyz")
    vb = lambda k: tuple(int(math.floor(before[c][k] / dv)) for c in "uvw")
    partners = {}
    for k2 in gone:
        cands = [k1 for k1 in keepers if cell(k1) == cell(k2) and vb(k1) == vb(k2) and
                 abs(before["q"][k1] + before["q"][k2] - p["q"][k1]) < 1e-18 and before["id"][k1] < before["id"][k2]]
        assert cands, "merged particle without a partner in its cell and velocity bin"
        partners[k2] = cands
    for k2, cands in partners.items():
        k1 = cands[0]
        q1, q2 = before["q"][k1], before["q"][k2]
        dv2 = sum((before[c][k1] - before[c][k2]) ** 2 for c in "uvw")
        lost += q1 * q2 / (q1 + q2) * dv2
    assert abs((E0 - E1) - lost) < 1e-12 * E0


def test_coalesce_hand_worked_cell():
    """Four particles in one cell; bins of width 1: (0,0,0) ids 5, 9; (1,0,0) id 7;
    (0,0,0) id 12.  Sorted: [5 (0,0,0)], [9 (0,0,0)], [12 (0,0,0)], [7 (1,0,0)] by
    bins then id -> merge (5, 9); then 12 and 7 differ -> m = 1 with frac 0.5 -> 2."""
    g = O.make_grid((1, 1, 1), (1.0, 1.0, 1.0), bc=(1, 1, 1), dt=0.5)
    p = {"x": np.array([0.1, 0.5, 0.7, 0.3]), "y": np.array([0.2, 0.2, 0.9, 0.4]), "z": np.array([0.3, 0.8, 0.1, 0.5]),
         "u": np.array([0.25, 1.5, 0.5, 0.75]), "v": np.array([0.5, 0.25, 0.75, 0.125]),
         "w": np.array([0.0, 0.5, 0.25, 0.5]), "q": np.array([1.0, 2.0, 3.0, 1.0]),
         "id": np.array([5, 7, 9, 12], dtype=np.int64)}
    st = np.zeros(4, dtype=np.int8)
    m = O.coalesce(g, p, st, 1.0, 0.5)
    assert m == 1
    assert list(st) == [O.ALIVE, O.ALIVE, O.MERGED, O.ALIVE]
    # keeper id 5 (slot 0) = charge-weighted mean of ids 5 (q 1) and 9 (q 3)
    assert p["q"][0] == 4.0
    np.testing.assert_allclose([p["x"][0], p["u"][0], p["w"][0]],
                               [(0.1 + 3 * 0.7) / 4, (0.25 + 3 * 0.5) / 4, (0.0 + 3 * 0.25) / 4], rtol=1e-15)


def test_coalesce_overfull_cell_and_wide_bins_hand_worked():
    """R31 / PAPER.md:243 ("in cells with an excessive number of particles"): no
    cell-size or velocity-range limit.  One cell with 2000 particles, ids 0..1999,
    u = (id % 2) + 1/2 (dv = 1: even ids in bin 0, odd ids in bin 1), frac = 1/2
    -> m = 1000 merges: the sorted list is [0, 2, ..., 1998 | 1, 3, ..., 1999], so
    the pairs are (0,2), (4,6), ..., (1996,1998) then (1,3), ..., (1997,1999) --
    every id = 2 mod 4 or 3 mod 4 is merged into id - 2.  A second cell holds
    two particles at u = 3e12 and 3e12 + 0.5 (same bin, floor = 3e12, far beyond
    any packed-key range) and one at -7e15 (own bin): frac 0.5 of 3 -> 1 merge."""
    g = O.make_grid((2, 1, 1), (2.0, 1.0, 1.0), bc=(1, 1, 1), dt=0.5)
    n = 2000
    ids = np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(4)
    p = {"x": rng.uniform(0.01, 0.99, n), "y": rng.uniform(0.01, 0.99, n), "z": rng.uniform(0.01, 0.99, n),
         "u": (ids % 2) + 0.5, "v": np.full(n, 0.25), "w": np.full(n, 0.75), "q": np.full(n, 1.0), "id": ids}
    wide = {"x": np.array([1.5, 1.25, 1.75]), "y": np.array([0.5, 0.5, 0.5]), "z": np.array([0.5, 0.5, 0.5]),
            "u": np.array([3e12, 3e12 + 0.5, -7e15]), "v": np.zeros(3), "w": np.zeros(3), "q": np.array([1.0, 3.0, 1.0]),
            "id": np.array([5000, 5001, 5002], dtype=np.int64)}
    P = {k: np.ascontiguousarray(np.concatenate([p[k], wide[k]])) for k in p}
    st = np.zeros(n + 3, dtype=np.int8)
    m = O.coalesce(g, P, st, 1.0, 0.5)
    assert m == 1000 + 1
    merged = set(np.nonzero(st == O.MERGED)[0].tolist())
    want = {i for i in range(n) if i % 4 in (2, 3)} | {n + 1}
    assert merged == want
    for i in range(0, n, 4):
        for k in (i, i + 1):
            assert P["q"][k] == 2.0 and P["u"][k] == p["u"][k]
            assert P["x"][k] == (p["x"][k] + p["x"][k + 2]) / 2
    assert P["q"][n] == 4.0 and P["u"][n] == (3e12 + 3 * (3e12 + 0.5)) / 4
