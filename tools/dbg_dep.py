"""Debug: GPU moments vs the oracle deposit of the GPU's own particles (C1, 1 cycle)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_2507_20719_b200 import inputs as I, pic
import parity_util as PU
import oracle as O
w = I.c1()
parts = I.make_species(w, device="cpu")
cap = [int(p["x"].numel() * 1.25) + 64 for p in parts]
cfg = pic.make_config(w, capacity=cap, ghost=2, kernel=pic.KERNEL_TILED)
ctx = pic.Context(cfg)
for s, p in enumerate(parts):
    ctx.set_particles(s, {k: v.cuda() for k, v in p.items()})
lo, EB = I.field_window(w, 2, device="cpu")
ctx.set_fields(EB.cuda())
for cyc in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    ctx.cycle()
print("stats", ctx.sync())
g = PU.oracle_grid(w)
for s in range(2):
    gp = {k: v.cpu().numpy() for k, v in ctx.get_particles(s).items()}
    gm = ctx.get_moments(s).cpu().numpy()
    m2, a2 = O.moments(g, {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in gp.items() if k != "id"}, None)
    print("species", s, "gm", gm.shape, "oracle", m2.shape, "n", len(gp["x"]))
    d = np.abs(gm - m2)
    for comp in range(10):
        r = d[comp] / np.maximum(a2[comp], 1e-300)
        print(comp, "sum gpu %.6e orc %.6e" % (gm[comp].sum(), m2[comp].sum()), "max ratio %.3e" % r.max(), "bad nodes", int((r > 1e-10).sum()), "of", r.size)
    r = d[0] / np.maximum(a2[0], 1e-300)
    idx = np.argwhere(r > 1e-10)[:8]
    for i in idx:
        print("  node", i, gm[0][tuple(i)], m2[0][tuple(i)])
