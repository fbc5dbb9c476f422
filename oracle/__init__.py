"""CPU oracle of the particle half of the implicit-moment PIC cycle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``libpic`` and ``paper_2507_20719_b200``) never
imports it, and it imports nothing from the product path.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, ``-O2
-ffp-contract=off``); this module only builds it with gcc and marshals numpy
arrays.  Passages followed: Eq. 2 for the mover, Eq. 3
 for the moments; readings R1..R23 in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

PERIODIC, OPEN = 0, 1
ALIVE, REMOVED, BAD, MERGED = 0, 1, 2, 3


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (no FMA contraction), and the
    same source with OpenMP into liboracle_omp.so (all-cores timing only)."""
    for lib, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
            tmp = lib + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                                   "-fPIC", "-shared"] + extra + ["-o", tmp, _SRC, "-lm"])
            os.replace(tmp, lib)
    return _LIB


class Grid(C.Structure):
    _fields_ = [("ncell", C.c_int64 * 3), ("len", C.c_double * 3), ("bc", C.c_int32 * 3),
                ("dt", C.c_double), ("c", C.c_double),
                ("planet_center", C.c_double * 3), ("planet_radius", C.c_double)]


class Field(C.Structure):
    _fields_ = [("lo", C.c_int64 * 3), ("n", C.c_int64 * 3), ("EB", C.POINTER(C.c_double))]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P = C.POINTER
        d = P(C.c_double)
        lib.oracle_sample.argtypes = [P(Grid), P(Field), d, d]
        lib.oracle_sample.restype = C.c_int
        lib.oracle_mover.argtypes = [P(Grid), P(Field), C.c_double, C.c_int, C.c_int64,
                                     d, d, d, d, d, d, P(C.c_int8)]
        lib.oracle_mover.restype = C.c_int64
        lib.oracle_mover_ex.argtypes = [P(Grid), P(Field), C.c_double, C.c_int, C.c_int, C.c_int64,
                                        d, d, d, d, d, d, P(C.c_int8)]
        lib.oracle_mover_ex.restype = C.c_int64
        lib.oracle_moments.argtypes = [P(Grid), C.c_int64, d, d, d, d, d, d, d, P(C.c_int8), d, d]
        lib.oracle_moments.restype = C.c_int64
        lib.oracle_node_counts.argtypes = [P(Grid), P(C.c_int64)]
        lib.oracle_implicit_sources.argtypes = [P(Grid), C.c_int, d, P(d), d, d, d, d]
        lib.oracle_implicit_sources.restype = None
        lib.oracle_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32)]
        lib.oracle_philox4x32_10.restype = None
        lib.oracle_inject.argtypes = [P(Grid), P(Field), C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint32,
                                      C.c_uint32, C.c_int64, C.c_int, C.c_double, d, C.c_double, C.c_int64,
                                      d, d, d, d, d, d, d, P(C.c_int64)]
        lib.oracle_inject.restype = C.c_int64
        lib.oracle_split.argtypes = [P(Grid), C.c_int, C.c_int64, C.c_int64, d, d, d, d, d, d, d,
                                     P(C.c_int64), P(C.c_int8), C.c_double, C.c_double, C.c_uint32, C.c_uint32,
                                     C.c_int64]
        lib.oracle_split.restype = C.c_int64
        lib.oracle_coalesce.argtypes = [P(Grid), C.c_int64, d, d, d, d, d, d, d, P(C.c_int64), P(C.c_int8),
                                        C.c_double, C.c_double]
        lib.oracle_coalesce.restype = C.c_int64
        lib.oracle_child_id.argtypes = [C.c_int64, C.c_int64]
        lib.oracle_child_id.restype = C.c_int64
        lib.oracle_bin_velocities.argtypes = [C.c_int64, d, d, d, d, P(C.c_int8), C.c_int, C.c_double, d]
        lib.oracle_bin_velocities.restype = C.c_int64
        lib.oracle_fit_gmm.argtypes = [C.c_int, C.c_double, d, C.c_int, C.c_int, d, d, d]
        lib.oracle_fit_gmm.restype = C.c_int
        _lib = lib
    return _lib


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_grid(ncell, length, bc=(PERIODIC,) * 3, dt=0.5, c=1.0,
              planet_center=(0.0, 0.0, 0.0), planet_radius=0.0) -> Grid:
    g = Grid()
    for d in range(3):
        g.ncell[d] = int(ncell[d])
        g.len[d] = float(length[d])
        g.bc[d] = int(bc[d])
        g.planet_center[d] = float(planet_center[d])
    g.dt, g.c, g.planet_radius = float(dt), float(c), float(planet_radius)
    return g


class FieldWindow:
    """E,B node window: global node indices [lo, lo+n) per axis, EB[k][j][i][6]."""

    def __init__(self, lo, EB: np.ndarray):
        EB = np.ascontiguousarray(EB, dtype=np.float64)
        assert EB.ndim == 4 and EB.shape[3] == 6
        self.EB = EB
        self.lo = tuple(int(v) for v in lo)
        self.n = (EB.shape[2], EB.shape[1], EB.shape[0])
        f = Field()
        for d in range(3):
            f.lo[d] = self.lo[d]
            f.n[d] = self.n[d]
        f.EB = _dptr(self.EB)
        self.c = f


def node_counts(g: Grid):
    out = (C.c_int64 * 3)()
    _load().oracle_node_counts(C.byref(g), out)
    return tuple(out)


def sample(g: Grid, F: FieldWindow, pos) -> np.ndarray:
    return sample_ex(g, F, pos)[0]


def sample_ex(g: Grid, F: FieldWindow, pos):
    """(E,B at pos, 1 if the R11 clamp to the window was applied else 0)."""
    p = np.ascontiguousarray(pos, dtype=np.float64)
    out = np.zeros(6)
    clamped = _load().oracle_sample(C.byref(g), C.byref(F.c), _dptr(p), _dptr(out))
    return out, int(clamped)


def mover(g: Grid, F: FieldWindow, qom: float, n_iter: int, parts: dict, status=None,
          relativistic: bool = False):
    """Push one species in place.  parts: dict of float64 arrays x y z u v w.
    relativistic: Eq. 2 with gamma (NEXT-1, readings R4/R5), else gamma == 1 (R3)."""
    n = len(parts["x"])
    if status is None:
        status = np.zeros(n, dtype=np.int8)
    for k in "xyzuvw":
        assert parts[k].dtype == np.float64 and parts[k].flags.c_contiguous
    bad = _load().oracle_mover_ex(C.byref(g), C.byref(F.c), float(qom), int(n_iter), int(bool(relativistic)), n,
                                  *[_dptr(parts[k]) for k in "xyzuvw"],
                                  status.ctypes.data_as(C.POINTER(C.c_int8)))
    return status, int(bad)


def moments(g: Grid, parts: dict, status=None, with_abs: bool = True):
    """Moments of one species: (mom[10][nz][ny][nx], absmom or None)."""
    nx, ny, nz = node_counts(g)
    mom = np.zeros((10, nz, ny, nx))
    am = np.zeros((10, nz, ny, nx)) if with_abs else None
    n = len(parts["x"])
    st = status.ctypes.data_as(C.POINTER(C.c_int8)) if status is not None else None
    out = _load().oracle_moments(C.byref(g), n, *[_dptr(parts[k]) for k in "xyzuvwq"], st,
                                 _dptr(mom), _dptr(am) if am is not None else None)
    if out:
        raise ValueError(f"{out} particles outside the grid in oracle.moments")
    return mom, am


_lib_omp = None


def _load_omp():
    """The OpenMP build (bench.py's all-cores cpu_baseline; never a parity checker)."""
    global _lib_omp
    if _lib_omp is None:
        build()
        lib = C.CDLL(_LIB_OMP)
        P = C.POINTER
        d = P(C.c_double)
        lib.oracle_omp_threads.restype = C.c_int
        lib.oracle_mover_par.argtypes = [P(Grid), P(Field), C.c_double, C.c_int, C.c_int, C.c_int64,
                                         d, d, d, d, d, d, P(C.c_int8)]
        lib.oracle_mover_par.restype = C.c_int64
        lib.oracle_moments_par.argtypes = [P(Grid), C.c_int64, d, d, d, d, d, d, d, P(C.c_int8), d]
        lib.oracle_moments_par.restype = C.c_int64
        _lib_omp = lib
    return _lib_omp


def omp_threads() -> int:
    return int(_load_omp().oracle_omp_threads())


def mover_par(g: Grid, F: FieldWindow, qom: float, n_iter: int, parts: dict, status=None,
              relativistic: bool = False):
    """`mover` on all host cores (OpenMP build; bit-identical results)."""
    n = len(parts["x"])
    if status is None:
        status = np.zeros(n, dtype=np.int8)
    bad = _load_omp().oracle_mover_par(C.byref(g), C.byref(F.c), float(qom), int(n_iter), int(bool(relativistic)),
                                       n, *[_dptr(parts[k]) for k in "xyzuvw"],
                                       status.ctypes.data_as(C.POINTER(C.c_int8)))
    return status, int(bad)


def moments_par(g: Grid, parts: dict, status=None):
    """`moments` on all host cores: per-thread node grids merged in thread order."""
    nx, ny, nz = node_counts(g)
    mom = np.zeros((10, nz, ny, nx))
    n = len(parts["x"])
    st = status.ctypes.data_as(C.POINTER(C.c_int8)) if status is not None else None
    out = _load_omp().oracle_moments_par(C.byref(g), n, *[_dptr(parts[k]) for k in "xyzuvwq"], st, _dptr(mom))
    if out:
        raise ValueError(f"{out} particles outside the grid in oracle.moments_par")
    return mom


def implicit_sources(g: Grid, qoms, moms, B: np.ndarray):
    """Eq. 5-6 (NEXT-2): chi[9][nz][ny][nx], rho_hat[nz][ny][nx], J_hat[3][nz][ny][nx]
    from per-species moments (oracle.moments layout) and node B[nz][ny][nx][3]."""
    nx, ny, nz = node_counts(g)
    S = len(moms)
    ms = [np.ascontiguousarray(m, dtype=np.float64) for m in moms]
    for m in ms:
        assert m.shape == (10, nz, ny, nx)
    Bc = np.ascontiguousarray(B, dtype=np.float64)
    assert Bc.shape == (nz, ny, nx, 3)
    q = np.ascontiguousarray(qoms, dtype=np.float64)
    arr = (C.POINTER(C.c_double) * S)(*[_dptr(m) for m in ms])
    chi = np.zeros((9, nz, ny, nx))
    rh = np.zeros((nz, ny, nx))
    jh = np.zeros((3, nz, ny, nx))
    _load().oracle_implicit_sources(C.byref(g), S, _dptr(q), arr, _dptr(Bc), _dptr(chi), _dptr(rh), _dptr(jh))
    return chi, rh, jh


def philox(counter, key):
    """Philox4x32-10 of one counter (4 x uint32) under key (2 x uint32)."""
    c = (C.c_uint32 * 4)(*[int(v) & 0xffffffff for v in counter])
    k = (C.c_uint32 * 2)(*[int(v) & 0xffffffff for v in key])
    _load().oracle_philox4x32_10(c, k)
    return [int(v) for v in c]


def inject(g: Grid, F: FieldWindow, species: int, qom: float, n_iter: int, seed: int, cycle: int, ppc: int,
           vth: float, drift, q: float, relativistic: bool = False) -> dict:
    """NEXT-3 inflow injection (reading R28): the particles that enter through the
    x = 0 face this cycle, after their first push (dict of arrays incl. int64 id)."""
    cap = int(g.ncell[1] * g.ncell[2] * ppc)
    out = {k: np.zeros(cap) for k in "xyzuvwq"}
    ids = np.zeros(cap, dtype=np.int64)
    dr = np.ascontiguousarray(drift, dtype=np.float64)
    n = _load().oracle_inject(C.byref(g), C.byref(F.c), int(species), float(qom), int(n_iter), int(bool(relativistic)),
                              seed & 0xffffffff, (seed >> 32) & 0xffffffff, int(cycle), int(ppc), float(vth), _dptr(dr),
                              float(q), cap, *[_dptr(out[k]) for k in "xyzuvwq"],
                              ids.ctypes.data_as(C.POINTER(C.c_int64)))
    if n < 0:
        raise ValueError("injection needs an open x axis")
    res = {k: a[:n].copy() for k, a in out.items()}
    res["id"] = ids[:n].copy()
    return res


def split(g: Grid, species: int, parts: dict, status, p_split: float, eps: float, seed: int, cycle: int):
    """NEXT-3 splitting (reading R30): returns (parts, status) with the children appended."""
    n = len(parts["x"])
    cap = 2 * n + 1
    P = {k: np.zeros(cap) for k in "xyzuvwq"}
    ids = np.zeros(cap, dtype=np.int64)
    st = np.zeros(cap, dtype=np.int8)
    for k in "xyzuvwq":
        P[k][:n] = parts[k]
    ids[:n] = parts["id"]
    st[:n] = status
    m = _load().oracle_split(C.byref(g), int(species), n, cap, *[_dptr(P[k]) for k in "xyzuvwq"],
                             ids.ctypes.data_as(C.POINTER(C.c_int64)), st.ctypes.data_as(C.POINTER(C.c_int8)),
                             float(p_split), float(eps), seed & 0xffffffff, (seed >> 32) & 0xffffffff, int(cycle))
    out = {k: P[k][:m].copy() for k in "xyzuvwq"}
    out["id"] = ids[:m].copy()
    return out, st[:m].copy()


def coalesce(g: Grid, parts: dict, status, dv: float, frac: float) -> int:
    """NEXT-3 coalescence (reading R31), in place; merged particles get status MERGED."""
    n = len(parts["x"])
    for k in "xyzuvwq":
        assert parts[k].dtype == np.float64 and parts[k].flags.c_contiguous
    return int(_load().oracle_coalesce(C.byref(g), n, *[_dptr(parts[k]) for k in "xyzuvwq"],
                                       parts["id"].ctypes.data_as(C.POINTER(C.c_int64)),
                                       status.ctypes.data_as(C.POINTER(C.c_int8)), float(dv), float(frac)))


def child_id(parent: int, cycle: int) -> int:
    return int(_load().oracle_child_id(int(parent), int(cycle)))


def bin_velocities(parts: dict, status, B: int, vmax: float):
    """NEXT-4 velocity histogram (reading R32): (hist[B][B][B] as [bz][by][bx], clipped)."""
    n = len(parts["u"])
    h = np.zeros((B, B, B))
    st = status.ctypes.data_as(C.POINTER(C.c_int8)) if status is not None else None
    c = _load().oracle_bin_velocities(n, *[_dptr(np.ascontiguousarray(parts[k], dtype=np.float64)) for k in "uvwq"],
                                      st, int(B), float(vmax), _dptr(h))
    return h, int(c)


def fit_gmm(hist: np.ndarray, vmax: float, M: int, n_em: int):
    """NEXT-4 EM fit (reading R33): (alpha[M], mu[M][3], sigma[M][6] as xx xy xz yy yz zz)."""
    B = hist.shape[0]
    h = np.ascontiguousarray(hist, dtype=np.float64)
    a, mu, sg = np.zeros(M), np.zeros((M, 3)), np.zeros((M, 6))
    rc = _load().oracle_fit_gmm(int(B), float(vmax), _dptr(h), int(M), int(n_em), _dptr(a), _dptr(mu), _dptr(sg))
    if rc != 0:
        raise ValueError("fewer occupied bins than components")
    return a, mu, sg
