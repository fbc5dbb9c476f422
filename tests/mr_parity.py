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

import slab_parity as SP  # noqa: E402
from paper_2507_20719_b200 import decomp, inputs as I, pic  # noqa: E402


def run_case(name, w, cycles, kernel, transport, rank, world, inject=None, orc_cache=None, graph=False):
    bounds = decomp.uniform_bounds(w.ncell[0], world)
    lo, hi = bounds[rank], bounds[rank + 1]
    parts_all, per_rank = SP.split_inputs(w, bounds)
    mine = per_rank[rank]
    wr = w.with_slab(lo, hi)
    nid = decomp.broadcast_nccl_id(pic.pic_nccl_id)
    cfg = pic.make_config(wr, rank=rank, nranks=world, capacity=SP.capacity(parts_all), ghost=2, kernel=kernel,
                          transport=transport)
    ctx = pic.Context(cfg, nccl_id=nid, stream=torch.cuda.Stream() if graph else None)
    ctx.set_graph(graph)
    assert ctx.transport == transport
    mine = [{k: v.cuda() for k, v in p.items()} for p in mine]
    torch.cuda.synchronize()          # torch's copies before libpic's stream reads them
    for s, p in enumerate(mine):
        ctx.set_particles(s, p)
        if inject:
            ctx.set_injection(s, inject["ppc"], w.species[s].vth, inject["drift"], float(parts_all[s]["q"][0]),
                              500 + s)
    _, EB = I.field_window(wr, 2, device="cpu")
    torch.cuda.synchronize()
    ctx.set_fields(EB.cuda())
    torch.cuda.synchronize()
    dist.barrier()           # every rank is set up before the first collective cycle
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
    key = (name, cycles)
    if orc_cache is None or key not in orc_cache:
        orc = SP.oracle_reference(w, parts_all, cycles, inject)
        if orc_cache is not None:
            orc_cache[key] = orc
    orc = orc_cache[key] if orc_cache is not None else orc
    return SP.check_union(name, w, gathered, orc, kernel=kernel, transport=transport, world=world)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--long", type=int, default=0,
                    help="only C1r for this many cycles, replayed from CUDA graphs over the peer transport")
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
    if args.long:
        # many replays of the same graphs: the device-side barrier epochs, the
        # peer receive buffers and the forward rounds over a long run
        res = run_case("c1r-long", I.c1(randomized=True), args.long, pic.KERNEL_TILED, pic.TRANSPORT_PEER, rank,
                       world, orc_cache={}, graph=True)
        if rank == 0:
            all_ok, reports = res
            for r in reports:
                r["graph"] = True
        cases = []
    inj_case = ("c4inj", I.c4(ncell=(32, 16, 16), ppc=8), 3, {"ppc": 8, "drift": (0.15, 0.0, 0.0)})
    orc_cache = {}
    for transport in (pic.TRANSPORT_PEER, pic.TRANSPORT_NCCL) if cases else ():
        for kernel in (pic.KERNEL_TILED, pic.KERNEL_BASIC):
            for name, w, cyc, *inj in cases + [inj_case]:
                res = run_case(name, w, cyc, kernel, transport, rank, world, inject=inj[0] if inj else None,
                               orc_cache=orc_cache)
                if rank == 0:
                    ok, reps = res
                    all_ok &= ok
                    reports += reps
    # whole cycles replayed from CUDA graphs over the peer transport (device-side
    # barrier epochs advance on every replay)
    for name, w, cyc, *inj in cases[:2]:
        res = run_case(name, w, cyc + 2, pic.KERNEL_TILED, pic.TRANSPORT_PEER, rank, world, orc_cache=orc_cache,
                       graph=True)
        if rank == 0:
            ok, reps = res
            for r in reps:
                r["graph"] = True
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
