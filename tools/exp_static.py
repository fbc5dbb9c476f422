"""Experiment: kernel times of the C2 step with the normal time step and with a
tiny one (no particle changes cell, so every gather through perm is contiguous).
The difference bounds what a physically sorted store could gain."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_20719_b200 import inputs as I, pic

def run(dt_scale):
    w = I.c2(ppc=125)
    w.dt = w.dt * dt_scale
    parts = I.make_species(w, device="cuda")
    cap = [int(p["x"].numel() * 1.08) + 65536 for p in parts]
    ctx = pic.Context(pic.make_config(w, capacity=cap))
    for s, p in enumerate(parts):
        ctx.set_particles(s, p)
    ctx.set_fields(I.field_window(w, 2, device="cuda")[1])
    for _ in range(4):
        ctx.cycle()
    ctx.sync()
    ctx.profile(True)
    for _ in range(5):
        ctx.cycle()
    prof = ctx.profile_read()
    ctx.profile(False)
    ctx.close()
    return {k: round(v[0] / 5, 4) for k, v in prof.items()}

for sc in (1.0, 1e-9, 1.0):
    print(sc, json.dumps(run(sc)), flush=True)
