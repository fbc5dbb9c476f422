"""Parity report: max error ratio (error / bound) of the CUDA path against the
oracle per configuration, kernel family and species (SURVEY.md §8(c) c.5:
"report the max error ratio, not just pass/fail").  Runs on one GPU:

    python tools/parity_report.py profiles/r01_parity_report.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import parity_util as PU  # noqa: E402
from paper_2507_20719_b200 import inputs as I, pic  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402


def main(out):
    cases = [("c1", I.c1(), 5), ("c1r", I.c1(randomized=True), 5), ("c1rel", I.c1rel(), 4),
             ("c2/8", I.c2(nx_per_rank=16, ppc=27), 3), ("c3 24^3", I.c3(n_per_rank=24, ppc=8), 3),
             ("c4 32x16x16", I.c4(ncell=(32, 16, 16), ppc=8), 4),
             ("c5 64x32x32", I.c5(ncell=(64, 32, 32), wind_ppc=4, inner_ppc=1, planet_ppc=32), 3)]
    rows = []
    for name, w, cyc in cases:
        parts = I.make_species(w, device="cpu")
        orc = PU.run_oracle(w, parts, cyc)
        g = PU.oracle_grid(w)
        for kernel, kname in ((pic.KERNEL_TILED, "tiled"), (pic.KERNEL_BASIC, "basic")):
            gpu, stats = run_gpu(w, parts, cyc, kernel)
            for s, sp in enumerate(w.species):
                rep = {"config": name, "kernel": kname, "species": sp.name, "cycles": cyc}
                okp = PU.compare_particles(w, sp, gpu[s][0], orc[s][0], orc[s][1], rep)
                okm = PU.compare_moments(gpu[s][1], orc[s][2], orc[s][3], rep)
                gp = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in gpu[s][0].items() if k != "id"}
                m2, a2 = O.moments(g, gp, None)
                r2 = {}
                PU.compare_moments(gpu[s][1], m2, a2, r2)
                rep["deposit_only_mom_ratio"] = r2.get("mom_ratio")
                rep["pass"] = bool(okp and okm)
                rows.append(rep)
                print(json.dumps(rep), flush=True)
    summary = {"what": "max error / bound per case (bounds: positions 1e-12 L, velocities 1e-12 max(|v|, v_th), "
                       "moments 1e-10 x sum|contributions|); pass = every ratio <= 1",
               "all_pass": all(r["pass"] for r in rows), "rows": rows}
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "parity_report.json")
