"""Decomposition-invariance harness (P14) shared by the multi-rank parity runs:
tests/mr_parity.py (one process per GPU, peer / NCCL transports) and
tests/test_gpu_loopback.py (the P slab contexts of one process on one GPU,
loopback transport).

The global inputs are drawn once (independent of the slab split), each rank
gets the particles of its x-slab, runs the cycle through the C ABI, and the
union of the slabs is compared with the single-process CPU oracle: particles
by id (positions, velocities, charge), moments per node within R19, and the
NEXT-2 sources two-level (the oracle fed with the union of the GPU moments).

Test infrastructure: imports the oracle; never imported by the product path.
"""
from __future__ import annotations

import numpy as np
import torch

import parity_util as PU
from paper_2507_20719_b200 import decomp, inputs as I


def split_inputs(w: I.Workload, bounds):
    """Global particles (CPU) and the per-rank subsets of the x-slabs (R21)."""
    parts_all = I.make_species(w.with_slab(0, w.ncell[0]), device="cpu")
    per_rank = []
    for r in range(len(bounds) - 1):
        mine = []
        for p in parts_all:
            cx = torch.floor(p["x"] / w.delta[0]).to(torch.int64)
            own = decomp.owner_of_cells(cx, bounds) == r
            mine.append({k: v[own].contiguous() for k, v in p.items()})
        per_rank.append(mine)
    return parts_all, per_rank


def capacity(parts_all):
    return [int(p["x"].numel() * 1.5) + 4096 for p in parts_all]


def oracle_reference(w: I.Workload, parts_all, cycles: int, inject=None):
    """Oracle state after `cycles` cycles of the whole (undecomposed) domain:
    [(parts, status, moments, absmoments)] per species; with `inject`, the
    NEXT-3 inflow of every cycle is appended as the GPU appends it (R28)."""
    if not inject:
        return PU.run_oracle(w.with_slab(0, w.ncell[0]), parts_all, cycles)
    import oracle as O
    wf = w.with_slab(0, w.ncell[0])
    g, F = PU.oracle_grid(wf), PU.oracle_field(wf, 2)
    orc = []
    for s, sp in enumerate(w.species):
        P = PU.to_numpy_parts(parts_all[s])
        st = np.zeros(len(P["x"]), dtype=np.int8)
        for c in range(cycles):
            st, _ = O.mover(g, F, sp.qom, w.n_iter, P, st)
            new = O.inject(g, F, s, sp.qom, w.n_iter, 500 + s, c, inject["ppc"], sp.vth, inject["drift"],
                           float(parts_all[s]["q"][0]))
            P = {k: np.concatenate([P[k], new[k]]) for k in P}
            st = np.concatenate([st, np.zeros(len(new["x"]), dtype=np.int8)])
        mom, am = O.moments(g, P, st)
        orc.append((P, st, mom, am))
    return orc


def check_union(name, w: I.Workload, gathered, orc, *, kernel, transport, world):
    """gathered[r] = ([(particles, moments)] per species, stats, sources or None)
    of rank r.  Returns (ok, reports)."""
    reps = []
    ok = True
    for s, sp in enumerate(w.species):
        gp = {k: np.concatenate([gathered[r][0][s][0][k] for r in range(world)]) for k in gathered[0][0][s][0]}
        gm = np.concatenate([gathered[r][0][s][1] for r in range(world)], axis=3)
        rep = {"case": name, "kernel": kernel, "transport": transport, "species": sp.name, "world": world,
               "sent": sum(g[1]["sent"] for g in gathered), "received": sum(g[1]["received"] for g in gathered),
               "removed": sum(g[1]["removed"] for g in gathered)}
        okp = PU.compare_particles(w, sp, gp, orc[s][0], orc[s][1], rep)
        okm = PU.compare_moments(gm, orc[s][2], orc[s][3], rep)
        rep["ok"] = bool(okp and okm)
        ok &= rep["ok"]
        reps.append(rep)
    if gathered[0][2] is not None:
        # two-level: the sources over the union of slabs vs the oracle fed with
        # the union of the GPU moments
        import oracle as O
        gms = [np.concatenate([gathered[r][0][s][1] for r in range(world)], axis=3) for s in range(len(w.species))]
        got = [np.concatenate([gathered[r][2][i] for r in range(world)], axis=-1) for i in range(3)]
        G = 2
        _, EB = I.field_window(w.with_slab(0, w.ncell[0]), G)
        nz, ny, nx = gms[0].shape[1:]
        Bn = EB[G:G + nz, G:G + ny, G:G + nx, 3:6].numpy()
        want = O.implicit_sources(PU.oracle_grid(w), [sp.qom for sp in w.species], gms, Bn)
        okS = all(np.allclose(a, b, rtol=0, atol=1e-12 * np.abs(b).max()) for a, b in zip(got, want))
        reps.append({"case": name, "kernel": kernel, "transport": transport, "world": world,
                     "sources_ok": bool(okS),
                     "sources_err": [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(got, want)]})
        ok &= okS
    return ok, reps
