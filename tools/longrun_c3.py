"""Production-length stability check at BASELINE's full C3 size on one GPU
(not a test: ~1 min of GPU time).  906 M particles, periodic, CUDA-graph
cycles: after CYCLES cycles every species still holds all its particles, the
ids are the same multiset (count, sum and sum of squares mod 2^64 of the ids,
before and after), sum_g rho_g V = sum_p q_p (P8), and the device counters
report no far-flyer, overflow or non-finite value.

    python tools/longrun_c3.py [--cycles 500] [--out report.json]
"""
import argparse
import json
import os
import sys
import time
import types

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2507_20719_b200 import inputs as I, pic  # noqa: E402

MASK = (1 << 64) - 1


def id_digest(ids):
    """(count, sum, sum of squares) of int64 ids, mod 2^64 (a permutation keeps all three)."""
    x = ids.to(torch.int64)
    return int(x.numel()), int(x.sum().item()) & MASK, int((x * x).sum().item()) & MASK


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=500)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    args = types.SimpleNamespace(config="c3", strong=False, ppc=0, c3_cells=192, relativistic=False, balance=1)
    w, desc = bench.workload(args, 1, 0)
    ub = I.species_upper_counts(w)
    stream = torch.cuda.Stream()
    ctx = pic.Context(pic.make_config(w, capacity=[int(n * 1.02) + 65536 for n in ub], ghost=2), stream=stream)
    before = [[0, 0, 0] for _ in w.species]
    qsum0 = [0.0 for _ in w.species]
    for _, _, parts in I.iter_species_chunks(w, 64_000_000, device="cuda"):
        torch.cuda.synchronize()
        for s, p in enumerate(parts):
            ctx.add_particles(s, p)
            n, s1, s2 = id_digest(p["id"])
            before[s] = [before[s][0] + n, (before[s][1] + s1) & MASK, (before[s][2] + s2) & MASK]
            qsum0[s] += float(p["q"].sum().item())
        del parts
    torch.cuda.empty_cache()
    _, EB = I.field_window(w, 2, device="cuda")
    torch.cuda.synchronize()
    ctx.set_fields(EB)
    ctx.set_graph(True)
    t0 = time.time()
    for _ in range(a.cycles):
        ctx.cycle()
    stats = ctx.sync()
    secs = time.time() - t0
    V = w.delta[0] * w.delta[1] * w.delta[2]
    rep = {"workload": desc, "cycles": a.cycles, "seconds": secs, "stats": stats, "species": []}
    ok = stats["far"] == 0 and stats["overflow"] == 0 and stats["nonfinite"] == 0 and stats["removed"] == 0
    for s, sp in enumerate(w.species):
        n = ctx.count(s)
        # the ids and charges of the live particles (the other components are not copied)
        import ctypes as C
        ids = torch.empty(n, dtype=torch.int64, device="cuda")
        q = torch.empty(n, dtype=torch.float64, device="cuda")
        P7 = (C.c_void_p * 7)(*[q.data_ptr() if k == "q" else None for k in "xyzuvwq"])
        assert ctx.lib.pic_get_particles(ctx.h, s, P7, C.c_void_p(ids.data_ptr())) == pic.PIC_OK
        digest = list(id_digest(ids))
        qsum = float(q.sum().item())
        del ids, q
        torch.cuda.empty_cache()
        gm = ctx.get_moments(s)
        rho = float(gm[0].sum().item()) * V
        del gm
        torch.cuda.empty_cache()
        r = {"species": sp.name, "count_before": before[s][0], "count_after": n, "ids_same": digest == before[s],
             "q_sum_before": qsum0[s], "q_sum_after": qsum, "rho_sum_rel_err": abs(rho - qsum) / abs(qsum)}
        r["ok"] = bool(n == before[s][0] and digest == before[s] and r["rho_sum_rel_err"] <= 1e-11 and
                       abs(qsum - qsum0[s]) <= 1e-12 * abs(qsum0[s]))
        ok &= r["ok"]
        rep["species"].append(r)
    rep["ok"] = bool(ok)
    txt = json.dumps(rep, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)
    ctx.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
