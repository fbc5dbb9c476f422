"""Multi-rank GPU parity (run under torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \
        --master-port 29533 tests/mr_parity.py [--out report.json]

Each rank owns an x-slab of the same global inputs, runs the full cycle through
the C ABI (both transports: peer memory over NVLink and NCCL messages, for
ghost-plane sums + migration), and rank 0 compares the union of
all slabs with the single-process CPU oracle (decomposition invariance, P14).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import parity_util as PU  # noqa: E402
from paper_2507_20719_b200 import decomp, inputs as I, pic  # noqa: E402


def run_case(name, w, cycles, kernel, transport, rank, world, inject=None):
    bounds = decomp.uniform_bounds(w.ncell[0], world)
    lo, hi = bounds[rank], bounds[rank + 1]
    parts_all = I.make_species(w.with_slab(0, w.ncell[0]), device="cpu")
    mine = []
    for p in parts_all:
        cx = torch.floor(p["x"] / w.delta[0]).to(torch.int64)
        own = decomp.owner_of_cells(cx, bounds) == rank
        mine.append({k: v[own].contiguous() for k, v in p.items()})
    wr = w.with_slab(lo, hi)
    cap = [int(p["x"].numel() * 1.5) + 4096 for p in parts_all]
    nid = decomp.broadcast_nccl_id(pic.pic_nccl_id)
    cfg = pic.make_config(wr, rank=rank, nranks=world, capacity=cap, ghost=2, kernel=kernel, transport=transport)
    ctx = pic.Context(cfg, nccl_id=nid)
    assert ctx.transport == transport
    for s, p in enumerate(mine):
        ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
        if inject:
            ctx.set_injection(s, inject["ppc"], w.species[s].vth, inject["drift"], float(parts_all[s]["q"][0]),
                              500 + s)
    _, EB = I.field_window(wr, 2, device="cpu")
    ctx.set_fields(EB.cuda())
    for _ in range(cycles):
        ctx.cycle()
    stats = ctx.sync()
    local = []
    for s in range(len(w.species)):
        gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
        gm = ctx.get_moments(s).cpu().numpy()
        local.append((gp, gm))
    # NEXT-2 sources (collective with the peer transport)
    src = None
    if transport == pic.TRANSPORT_PEER:
        src = tuple(t.cpu().numpy() for t in ctx.implicit_sources())
    ctx.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, (local, stats, src))
    if rank != 0:
        return None
    if inject:
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
    else:
        orc = PU.run_oracle(w.with_slab(0, w.ncell[0]), parts_all, cycles)
    reps = []
    ok = True
    for s, sp in enumerate(w.species):
        gp = {k: np.concatenate([gathered[r][0][s][0][k] for r in range(world)]) for k in gathered[0][0][s][0]}
        gm = np.concatenate([gathered[r][0][s][1] for r in range(world)], axis=3)
        rep = {"case": name, "kernel": kernel, "transport": transport, "species": sp.name, "world": world,
               "sent": sum(g[1]["sent"] for g in gathered), "removed": sum(g[1]["removed"] for g in gathered)}
        okp = PU.compare_particles(w, sp, gp, orc[s][0], orc[s][1], rep)
        okm = PU.compare_moments(gm, orc[s][2], orc[s][3], rep)
        rep["ok"] = bool(okp and okm)
        ok &= rep["ok"]
        reps.append(rep)
    if transport == pic.TRANSPORT_PEER:
        # two-level: sources over the union of slabs vs the oracle fed with the
        # union of the GPU moments
        import oracle as O
        gms = [np.concatenate([gathered[r][0][s][1] for r in range(world)], axis=3) for s in range(len(w.species))]
        got = [np.concatenate([gathered[r][2][i] for r in range(world)], axis=-1) for i in range(3)]
        G = 2
        _, EB = I.field_window(w.with_slab(0, w.ncell[0]), G)
        nz, ny, nx = gms[0].shape[1:]
        Bn = EB[G:G + nz, G:G + ny, G:G + nx, 3:6].numpy()
        want = O.implicit_sources(PU.oracle_grid(w), [sp.qom for sp in w.species], gms, Bn)
        okS = all(np.allclose(a, b, rtol=0, atol=1e-12 * np.abs(b).max()) for a, b in zip(got, want))
        reps.append({"case": name, "kernel": kernel, "transport": transport, "sources_ok": bool(okS),
                     "sources_err": [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(got, want)]})
        ok &= okS
    return ok, reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    cases = [("c1r", I.c1(randomized=True), 4),
             ("c2s", I.c2(nx_per_rank=32, ppc=27), 3),
             ("c4s", I.c4(ncell=(32, 16, 16), ppc=8), 4),
             ("c5s", I.c5(ncell=(64, 32, 32), wind_ppc=2, inner_ppc=1, planet_ppc=16), 3)]
    all_ok, reports = True, []
    inj_case = ("c4inj", I.c4(ncell=(32, 16, 16), ppc=8), 3, {"ppc": 8, "drift": (0.15, 0.0, 0.0)})
    for transport in (pic.TRANSPORT_PEER, pic.TRANSPORT_NCCL):
        for kernel in (pic.KERNEL_TILED, pic.KERNEL_BASIC):
            for name, w, cyc, *inj in cases + [inj_case]:
                res = run_case(name, w, cyc, kernel, transport, rank, world, inject=inj[0] if inj else None)
                if rank == 0:
                    ok, reps = res
                    all_ok &= ok
                    reports += reps
    if rank == 0:
        txt = json.dumps({"ok": bool(all_ok), "reports": reports}, indent=1)
        print(txt)
        if args.out:
            with open(args.out, "w") as f:
                f.write(txt)
    okt = torch.tensor([1 if (rank != 0 or all_ok) else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    return 0 if okt.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
