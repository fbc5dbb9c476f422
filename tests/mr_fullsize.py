"""Multi-rank parity at full size ("a sub-slab sample at
full size"), run under torchrun with one rank per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29561 tests/mr_fullsize.py --config c4 [--out report.json]

The workload is bench.py's, built the way bench.py builds it (count-balanced
x-slabs for C4, each rank's slab drawn on its device sub-slab by sub-slab and
appended with pic_add_particles, peer transport, CUDA-graph cycles), for two
cycles.  The oracle cannot move 4.29e9 particles, so it checks samples one by
one: ~3000 particles per species by id (wherever they migrated) and 8 nodes
whose every contributor (the input particles within two cells, on whichever
rank they started) it moves and deposits; and Sum rho V over all ranks equals
the charge of all the GPU's particles (P8).  Rank 0 gathers and compares.
"""
import argparse
import json
import os
import sys
import types

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
import parity_util as PU  # noqa: E402
from paper_2507_20719_b200 import decomp, inputs as I, pic  # noqa: E402

CYCLES = 2
N_SAMPLE = 3000


def box_mask(p, node, w, half=2):
    m = torch.ones(p["x"].numel(), dtype=torch.bool, device=p["x"].device)
    for d, k in enumerate("xyz"):
        c = torch.floor(p[k] / w.delta[d])
        diff = c - float(node[d])
        if w.bc[d] == I.PERIODIC:
            diff = diff - w.ncell[d] * torch.round(diff / w.ncell[d])
        m &= (diff >= -half) & (diff <= half - 1)
    return m


def component(ctx, s, key, n):
    import ctypes as C
    out = torch.empty(n, dtype=torch.int64 if key == "id" else torch.float64, device="cuda")
    P7 = (C.c_void_p * 7)(*[out.data_ptr() if k == key else None for k in "xyzuvwq"])
    st = ctx.lib.pic_get_particles(ctx.h, s, P7, C.c_void_p(out.data_ptr()) if key == "id" else None)
    assert st == pic.PIC_OK, ctx.lib.pic_last_error(ctx.h)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    args = types.SimpleNamespace(config=a.config, strong=False, ppc=0, c3_cells=192, relativistic=False, balance=1)
    wr, desc = bench.workload(args, world, rank)
    lo, hi = wr.slab_or_all()
    wf = wr.with_slab(0, wr.ncell[0])
    ub = I.species_upper_counts(wr)
    cap = [int(n * 1.02) + 65536 for n in ub]
    nid = decomp.broadcast_nccl_id(pic.pic_nccl_id)
    stream = torch.cuda.Stream()
    ctx = pic.Context(pic.make_config(wr, rank=rank, nranks=world, capacity=cap, ghost=2), nccl_id=nid,
                      stream=stream)
    rng = np.random.default_rng(4242)
    nodes = [tuple(int(rng.integers(0, wr.ncell[d])) for d in range(3)) for _ in range(8)]
    total = sum(I.species_upper_counts(wf))
    p_pick = N_SAMPLE * len(wr.species) / total
    gen = torch.Generator(device="cuda").manual_seed(99 + rank)
    keep = [[] for _ in wr.species]
    for _, _, parts in I.iter_species_chunks(wr, 64_000_000, device="cuda"):
        torch.cuda.synchronize()
        for s, p in enumerate(parts):
            ctx.add_particles(s, p)
            m = torch.rand(p["x"].numel(), generator=gen, device="cuda") < p_pick
            for node in nodes:
                m |= box_mask(p, node, wr)
            keep[s].append({k: v[m].cpu() for k, v in p.items()})
        del parts
    torch.cuda.empty_cache()
    _, EB = I.field_window(wr, 2, device="cuda")
    torch.cuda.synchronize()
    ctx.set_fields(EB)
    ctx.set_graph(True)
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(CYCLES):
        ctx.cycle()
    stats = ctx.sync()
    del EB
    torch.cuda.empty_cache()
    V = wr.delta[0] * wr.delta[1] * wr.delta[2]
    # the kept inputs of every rank (sample + node contributors), on every rank
    kept = [{k: torch.cat([c[k] for c in keep[s]]) for k in keep[s][0]} for s in range(len(wr.species))]
    allkept = [None] * world
    dist.all_gather_object(allkept, kept)
    # GPU particles with the kept ids (wherever they migrated) and the owned moments at the nodes
    shape = ctx.moment_shape()
    found, node_vals, rho_ok = [], [], []
    for s in range(len(wr.species)):
        want = torch.from_numpy(np.sort(np.concatenate([allkept[r][s]["id"].numpy() for r in range(world)]))).cuda()
        n = ctx.count(s)
        gid = component(ctx, s, "id", n)
        pos = []
        for c0 in range(0, n, 100_000_000):
            ch = gid[c0:c0 + 100_000_000]
            j = torch.searchsorted(want, ch).clamp(max=want.numel() - 1)
            pos.append(torch.nonzero(want[j] == ch).flatten() + c0)
        pos = torch.cat(pos)
        f = {"id": gid[pos].cpu().numpy()}
        del gid
        qsum = 0.0
        for k in "xyzuvwq":
            arr = component(ctx, s, k, n)
            f[k] = arr[pos].cpu().numpy()
            if k == "q":
                qsum = float(arr.sum().item())
            del arr
        torch.cuda.empty_cache()
        found.append(f)
        gm = ctx.get_moments(s)
        rho_ok.append((float(gm[0].sum().item()) * V, qsum))
        vals = {}
        for node in nodes:
            if lo <= node[0] < lo + shape[0]:
                vals[node] = gm[:, node[2], node[1], node[0] - lo].cpu().numpy()
        node_vals.append(vals)
        del gm
        torch.cuda.empty_cache()
    gathered = [None] * world
    dist.all_gather_object(gathered, (found, node_vals, rho_ok, stats))
    ctx.close()
    ok = True
    if rank == 0:
        import oracle as O
        g, F = PU.oracle_grid(wf), PU.oracle_field(wf, 2)
        reports = []
        for s, sp in enumerate(wr.species):
            P = PU.to_numpy_parts({k: torch.cat([allkept[r][s][k] for r in range(world)]) for k in allkept[0][s]})
            st = np.zeros(len(P["x"]), dtype=np.int8)
            for _ in range(CYCLES):
                st, bad = O.mover(g, F, sp.qom, wr.n_iter, P, st)
                assert bad == 0
            gp = {k: np.concatenate([gathered[r][0][s][k] for r in range(world)]) for k in gathered[0][0][s]}
            rep = {"config": a.config, "world": world, "species": sp.name, "sampled": int(len(P["x"]))}
            okp = PU.compare_particles(wf, sp, gp, P, st, rep)
            mom, am = O.moments(g, P, st)
            worst = 0.0
            for node in nodes:
                gv = next(gathered[r][1][s][node] for r in range(world) if node in gathered[r][1][s])
                o, aa = mom[:, node[2], node[1], node[0]], am[:, node[2], node[1], node[0]]
                zero = aa == 0
                okz = bool(np.all(gv[zero] == 0.0))
                r_ = np.abs(gv - o) / np.where(zero, 1.0, PU.MOM_TOL * aa)
                worst = max(worst, float(np.where(zero, 0.0, r_).max()))
                ok &= okz
            rep["node_mom_ratio"] = worst
            # P8 over all particles and ranks: sum_g rho_g V = sum_p q_p (the ghost-plane sums
            # move a slab edge's deposits into the neighbour's planes, so per rank they differ)
            rs = sum(gathered[r][2][s][0] for r in range(world))
            qs = sum(gathered[r][2][s][1] for r in range(world))
            rep["rho_sum_rel_err"] = abs(rs - qs) / max(abs(qs), 1e-300)
            rep["ok"] = bool(okp and worst <= 1.0 and rep["rho_sum_rel_err"] <= 1e-11)
            ok &= rep["ok"]
            reports.append(rep)
        stats_all = [gathered[r][3] for r in range(world)]
        ok &= all(x["far"] == 0 and x["overflow"] == 0 and x["nonfinite"] == 0 for x in stats_all)
        txt = json.dumps({"ok": bool(ok), "workload": desc, "reports": reports, "stats": stats_all}, indent=1)
        print(txt)
        if a.out:
            with open(a.out, "w") as fo:
                fo.write(txt)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    return 0 if okt.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
