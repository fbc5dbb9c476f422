"""The all-cores build of the oracle (bench.py's cpu_baseline, SURVEY.md
§8(d.4)) computes what the single-threaded parity checker computes: the mover
bit for bit (particles are independent), the moments within R19 (per-thread
node grids merged in thread order only reassociate the sums)."""
import numpy as np

import oracle as O
import parity_util as PU
from paper_2507_20719_b200 import inputs as I


def test_omp_build_matches_reference_order():
    w = I.c1(randomized=True)
    parts = I.make_species(w)
    g, F = PU.oracle_grid(w), PU.oracle_field(w, 2)
    assert O.omp_threads() >= 1
    for s, sp in enumerate(w.species):
        A = PU.to_numpy_parts(parts[s])
        B = {k: v.copy() for k, v in A.items()}
        sa, ba = O.mover(g, F, sp.qom, 3, A)
        sb, bb = O.mover_par(g, F, sp.qom, 3, B)
        assert ba == bb == 0 and np.array_equal(sa, sb)
        for k in "xyzuvw":
            assert np.array_equal(A[k], B[k]), k
        mom, am = O.moments(g, A, sa)
        mp = O.moments_par(g, B, sb)
        assert np.all(np.abs(mp - mom) <= 1e-10 * am)
        assert np.all(mp[am == 0] == 0)
