#!/usr/bin/env python3
"""Small cases that launch every libpic kernel once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck; one tool per
run):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py

Covers mover_tiled_kernel / deposit_tiled_kernel (C1r), the basic family, the
order build, coalesce_kernel + coalesce_big_kernel (an overfull cell), split,
the GMM histogram + EM, the NEXT-2 source kernels, inflow injection (C4 clone,
open faces, planet) and the peer-transport kernels (send_leavers_peer in the
movers, arrive_kernel, ghost_pull_kernel) through a two-slab loopback pair.
Prints one line per case; exits non-zero on any libpic error.
"""
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_20719_b200 import decomp, inputs as I, pic  # noqa: E402


def small_c1r():
    w = I.c1(randomized=True)
    w.ncell = (8, 8, 8)
    w.length = (2.0, 2.0, 2.0)
    for sp in w.species:
        sp.ppc = 8
    return w


def run_single(w, kernel, cycles=2, extra=None):
    parts = I.make_species(w, device="cuda")
    ctx = pic.Context(pic.make_config(w, capacity=[int(p["x"].numel() * 2.5) + 2048 for p in parts], kernel=kernel))
    for s, p in enumerate(parts):
        ctx.set_particles(s, p)
    ctx.set_fields(I.field_window(w, 2, device="cuda")[1])
    for _ in range(cycles):
        ctx.cycle()
    if extra:
        extra(ctx, parts)
    stats = ctx.sync()
    ctx.close()
    return stats


def control_and_gmm(ctx, parts):
    n0 = [p["x"].numel() for p in parts]
    ctx.control(0, int(1.3 * n0[0]), 0.05, 0.1, 0.025, 3)          # split
    ctx.cycle()
    # an overfull cell for the unpacked coalescence path
    d = ctx.cfg.len[0] / ctx.cfg.ncell[0]
    n = 700
    big = {k: torch.full((n,), 1.5 * d, dtype=torch.float64, device="cuda") for k in "xyz"}
    big["x"] = big["x"] + torch.rand(n, device="cuda", dtype=torch.float64) * 0.4 * d
    for k in "uvw":
        big[k] = 0.01 * torch.randn(n, device="cuda", dtype=torch.float64)
    big["q"] = torch.full((n,), -1e-3, dtype=torch.float64, device="cuda")
    big["id"] = torch.arange(n, dtype=torch.int64, device="cuda") + (1 << 45)
    ctx.add_particles(0, big)
    ctx.control(0, int(0.7 * ctx.count(0)), 0.05, 0.1, 0.025, 3)   # coalesce
    ctx.cycle()
    ctx.gmm(0, 16, 0.25, 3, 10)
    ctx.implicit_sources()


def injection(ctx, parts):
    for s in range(len(parts)):
        ctx.set_injection(s, 4, 0.05, (0.1, 0.0, 0.0), float(parts[s]["q"][0].item()), 11 + s)
    for _ in range(2):
        ctx.cycle()


def loopback_pair():
    w = small_c1r()
    bounds = decomp.uniform_bounds(w.ncell[0], 2)
    parts_all = I.make_species(w, device="cpu")
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs = []
    for r in range(2):
        wr = w.with_slab(bounds[r], bounds[r + 1])
        cfg = pic.make_config(wr, rank=r, nranks=2, capacity=[p["x"].numel() + 4096 for p in parts_all],
                              transport=pic.TRANSPORT_LOOPBACK)
        ctx = pic.Context(cfg, stream=streams[r])
        dev = []
        for s, p in enumerate(parts_all):
            cx = torch.floor(p["x"] / w.delta[0]).to(torch.int64)
            own = decomp.owner_of_cells(cx, bounds) == r
            dev.append({k: v[own].contiguous().cuda() for k, v in p.items()})
        EB = I.field_window(wr, 2, device="cuda")[1]
        torch.cuda.synchronize()      # torch's work before libpic's stream reads it
        for s, p in enumerate(dev):
            ctx.set_particles(s, p)
        ctx.set_fields(EB)
        ctxs.append(ctx)
    pic.pic_loopback_link(ctxs)
    torch.cuda.synchronize()
    errs = []

    def body(r):
        try:
            with torch.cuda.stream(streams[r]):
                for _ in range(3):
                    ctxs[r].cycle()
                ctxs[r].sync()
                ctxs[r].implicit_sources()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    stats = [c.sync() for c in ctxs]
    for c in ctxs:
        c.close()
    if errs:
        raise errs[0]
    return stats


def main():
    torch.cuda.set_device(0)
    w = small_c1r()
    for kernel, name in ((pic.KERNEL_TILED, "tiled"), (pic.KERNEL_BASIC, "basic")):
        print(name, run_single(w, kernel), flush=True)
        print(name, "control+gmm+sources", run_single(w, kernel, 1, control_and_gmm), flush=True)
    w4 = I.c4(ncell=(16, 8, 8), ppc=4)
    print("c4 injection", run_single(w4, pic.KERNEL_TILED, 1, injection), flush=True)
    print("loopback", loopback_pair(), flush=True)
    print("sanitize_cases ok", flush=True)


if __name__ == "__main__":
    main()
