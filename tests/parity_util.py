"""Parity harness: run the oracle and the CUDA path on the same seeded inputs and
compare them with the north_star tolerances.

  positions   min-image per axis, |x_g - x_o| <= 1e-12 L_d
  velocities  |v_g - v_o|_inf <= 1e-12 max(|v_o|_2, v_th,s)
  removed     the same set (ids), except particles within 1e-12 L of a face
  moments     per node and component |g - o| <= 1e-10 A, A = sum |contributions|
              (R19; A = 0 => g must be exactly 0)

Test infrastructure: imports the oracle; never imported by the product path.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2507_20719_b200 import inputs as I

POS_TOL = 1e-12
VEL_TOL = 1e-12
MOM_TOL = 1e-10


def oracle_grid(w: I.Workload):
    return O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c, w.planet_center, w.planet_radius)


def oracle_field(w: I.Workload, ghost: int):
    lo, EB = I.field_window(w.with_slab(0, w.ncell[0]), ghost, device="cpu")
    return O.FieldWindow(lo, EB.numpy())


def to_numpy_parts(p):
    return {k: p[k].detach().cpu().numpy().astype(np.float64 if k != "id" else np.int64).copy()
            for k in ("x", "y", "z", "u", "v", "w", "q", "id")}


def run_oracle(w: I.Workload, species_parts, cycles: int, ghost: int = 2, n_iter=None):
    """Mover + moments for `cycles` cycles; returns (parts, status, moments, absmoments)
    per species after the last cycle (moments of the final state)."""
    g = oracle_grid(w)
    F = oracle_field(w, ghost)
    out = []
    for s, sp in enumerate(w.species):
        P = to_numpy_parts(species_parts[s])
        st = np.zeros(len(P["x"]), dtype=np.int8)
        for _ in range(cycles):
            st, bad = O.mover(g, F, sp.qom, n_iter or w.n_iter, P, st, relativistic=w.relativistic)
            assert bad == 0, "oracle flagged a bad particle"
        mom, am = O.moments(g, P, st)
        out.append((P, st, mom, am))
    return out


def compare_particles(w: I.Workload, sp: I.Species, gpu: dict, orc: dict, status, report: dict):
    """Compare GPU particles (live, any order) with oracle particles by id."""
    alive = status == O.ALIVE
    oid = orc["id"][alive]
    gid = gpu["id"]
    assert len(np.unique(gid)) == len(gid), "duplicate ids on the GPU"
    # removed-set check (flips within 1e-12 L of a face are tolerated)
    so, sg = set(oid.tolist()), set(gid.tolist())
    only_o, only_g = so - sg, sg - so
    face_flips = 0
    if only_o or only_g:
        pos_all = np.stack([orc["x"], orc["y"], orc["z"]], 1)
        idx_of = {int(i): k for k, i in enumerate(orc["id"])}
        for i in list(only_o) + list(only_g):
            k = idx_of[int(i)]
            x = pos_all[k]
            near = any(min(abs(x[d]), abs(x[d] - w.length[d])) <= POS_TOL * w.length[d] for d in range(3))
            if w.planet_radius > 0:
                r = np.linalg.norm(x - np.array(w.planet_center))
                near |= abs(r - w.planet_radius) <= POS_TOL * max(w.length)
            assert near, f"particle {i} alive on one side only, not near a face"
            face_flips += 1
    common = np.array(sorted(so & sg), dtype=np.int64)
    go = np.argsort(gid)
    gsorted = {k: gpu[k][go] for k in gpu}
    gi = np.searchsorted(gsorted["id"], common)
    oo = np.argsort(orc["id"])
    osorted = {k: orc[k][oo] for k in orc}
    oi = np.searchsorted(osorted["id"], common)
    worst_pos, worst_vel = 0.0, 0.0
    for d, k in enumerate("xyz"):
        L = w.length[d]
        diff = gsorted[k][gi] - osorted[k][oi]
        if w.bc[d] == I.PERIODIC:
            diff = diff - L * np.round(diff / L)
        worst_pos = max(worst_pos, float(np.max(np.abs(diff), initial=0.0)) / (POS_TOL * L))
    vo = np.stack([osorted[k][oi] for k in "uvw"], 1)
    vg = np.stack([gsorted[k][gi] for k in "uvw"], 1)
    scale = np.maximum(np.linalg.norm(vo, axis=1), sp.vth)
    err = np.max(np.abs(vg - vo), axis=1) / (VEL_TOL * scale)
    worst_vel = float(np.max(err, initial=0.0))
    qerr = float(np.max(np.abs(gsorted["q"][gi] - osorted["q"][oi]), initial=0.0))
    report.update(n=len(common), face_flips=face_flips, pos_ratio=worst_pos, vel_ratio=worst_vel, q_err=qerr)
    return worst_pos <= 1.0 and worst_vel <= 1.0 and qerr == 0.0


def compare_moments(gpu_mom: np.ndarray, orc_mom: np.ndarray, orc_abs: np.ndarray, report: dict):
    assert gpu_mom.shape == orc_mom.shape, (gpu_mom.shape, orc_mom.shape)
    err = np.abs(gpu_mom - orc_mom)
    bound = MOM_TOL * orc_abs
    zero = orc_abs == 0
    ok_zero = bool(np.all(gpu_mom[zero] == 0.0))
    ratio = np.where(zero, 0.0, err / np.where(zero, 1.0, bound))
    report.update(mom_ratio=float(ratio.max(initial=0.0)), mom_zero_ok=ok_zero)
    return ok_zero and float(ratio.max(initial=0.0)) <= 1.0
