#!/usr/bin/env python3
"""Bench: particle updates/s (mover + moments) of the implicit-moment PIC particle
path on 1..8 B200, and its fraction of the HBM roofline (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config c3] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A step is one full particle cycle through the C ABI (pic_mover, pic_moments,
pic_exchange) for every species of the workload.  The default workload is C3,
BASELINE.json configs[2] and the largest configuration that fits one GPU: the
weak-scaling cube of 192^3 cells per GPU, 2 species, 64 ppc (905,969,664
particles, a 136 GB store per GPU), x-slabs of 192 cells per rank with N GPUs.
`--config c2` is the GEM Harris sheet (configs[1]).  Inputs live in HBM and are
far larger than L2 (no flush needed).  Besides the HBM roofline of the dominant
kernel the line carries %fp64 (roofline_fp64) and the oracle timed on one host
core and on all of them (cpu_baseline).

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_ALG_PARTICLE = 104.0       # read x,v,q (56 B) + write x,v (48 B) per update


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5", "c4s", "c5s"])
    ap.add_argument("--impl", default="pic", choices=["pic", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 basic, 2 tiled")
    ap.add_argument("--transport", type=int, default=0, help="multi-GPU: 0 auto (peer memory), 1 NCCL, 2 peer")
    ap.add_argument("--relativistic", action="store_true", help="relativistic Eq. 2 (NEXT-1) on the same workload")
    ap.add_argument("--control", action="store_true", help="also time one particle-control split and coalescence pass (NEXT-3)")
    ap.add_argument("--gmm", action="store_true", help="also time the velocity binning + GMM fit of every species (NEXT-4)")
    ap.add_argument("--strong", action="store_true", help="c2/c3: fixed total problem (one GPU's) split over the N ranks")
    ap.add_argument("--balance", type=int, default=1, help="c4s/c5s with N>1: count-balanced slabs (1) or uniform (0)")
    ap.add_argument("--ghost", type=int, default=2)
    ap.add_argument("--ppc", type=int, default=0, help="override ppc (debug only)")
    ap.add_argument("--c3-cells", type=int, default=192,
                    help="c3: cells per GPU along each axis (192 = BASELINE configs[2]; smaller only for ncu clones)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle CPU time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: time the step as pic_cycle replayed from CUDA graphs where libpic allows it "
                         "(the per-kernel roofline then comes from a second, profiled pass of the same steps)")
    return ap.parse_args()


def workload(args, nranks, rank):
    from paper_2507_20719_b200 import inputs as I
    strong = getattr(args, "strong", False)
    if args.config == "c2":
        w = I.c2(scale_x=1 if strong else nranks, ppc=args.ppc or 125)
        per = 128 // nranks if strong else 128
        desc = ("C2 GEM double Harris sheet, 128x64x32 cells in total split into N x-slabs (strong scaling)" if strong else
                "C2 GEM double Harris sheet, 128x64x32 cells per GPU (x-slab weak scaling)") + \
            ", 2 species, 125 ppc, mass ratio 256, 3 PC iterations"
    elif args.config == "c3":
        n3 = args.c3_cells
        w = I.c3(nranks=1 if strong else nranks, ppc=args.ppc or 64, n_per_rank=n3)
        per = n3 // nranks if strong else n3
        desc = (f"C3 cube {n3}^3 cells in total split into N x-slabs (strong scaling)" if strong else
                f"C3 weak-scaling cube {n3}^3 cells per GPU") + ", 2 species, 64 ppc, 3 PC iterations" + \
            ("" if n3 == 192 else " (reduced clone for profiling, not BASELINE's size)")
    elif args.config == "c4":
        w = I.c4(ppc=args.ppc or 64)
        per = w.ncell[0] // nranks
        desc = ("C4 at full size: 512x256x256 cells (4.29e9 particles), open boundaries, absorbing planet, "
                "dipole + IMF, wind e-/p+ 64 ppc, removal only, 3 PC iterations (needs >= 4 GPUs)")
    elif args.config == "c5":
        w = I.c5()
        per = w.ncell[0] // nranks
        desc = ("C5 at full size: 512x256x256 cells, 4 species (wind e-/p+ 64/8 ppc, planetary e-/p+ "
                "round(256 exp(-(r-R)/2)) ppc), open boundaries, absorbing moon, 3 PC iterations (needs >= 4 GPUs)")
    elif args.config == "c4s":
        w = I.c4(ncell=(128 * nranks, 128, 128), ppc=args.ppc or 64)
        per = 128
        desc = ("C4 structure at 128^3 cells per GPU: open boundaries, absorbing planet, dipole + IMF, wind e-/p+ "
                "64 ppc, inflow injection of both species at x = 0 (NEXT-3), 3 PC iterations")
    elif args.config == "c5s":
        w = I.c5(ncell=(128 * nranks, 128, 128))
        per = 128
        desc = ("C5 structure at 128^3 cells per GPU: 4 species (wind e-/p+ 64 ppc outside the magnetosphere "
                "ellipsoid, 8 inside; planetary e-/p+ round(256 exp(-(r-R)/2)) ppc), open boundaries, absorbing moon")
    else:
        w = I.c1()
        per = 16 // nranks
        desc = "C1 16^3 periodic uniform Maxwellian, 2 species, 27 ppc (L2-resident; not a roofline config)"
    if args.relativistic:
        w.relativistic = True
        desc += "; relativistic Eq. 2 (NEXT-1)"
    if args.config in ("c4", "c5", "c4s", "c5s") and nranks > 1 and args.balance:
        # magnetosphere configs: slabs cut by the particle count per x-plane (H10)
        from paper_2507_20719_b200 import decomp
        b = decomp.balanced_bounds(I.plane_counts(w).tolist(), nranks, min_width=8)
        desc += "; count-balanced x-slabs"
        return w.with_slab(b[rank], b[rank + 1]), desc
    return w.with_slab(rank * per, (rank + 1) * per), desc


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons DURING the timed region.

    NVML is polled every ~2 ms from a thread (the GPU is matched by its PCI bus
    id, not by index), so even a 20 ms timed region gets a dozen samples;
    `nvidia-smi -lms 100` is the fallback when NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []          # (wall time, sm MHz, max sm MHz, set of reason names)
        self.proc = None
        self.nvml = None
        self.t0 = self.t1 = None
        self.stop = False

    def _open_nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = None
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.idx)
            h = N.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        except Exception:
            h = N.nvmlDeviceGetHandleByIndex(self.idx)
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        return N, h, bits, mx

    def _poll_nvml(self):
        N, h, bits, mx = self.nvml
        while not self.stop:
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((time.time(), float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            self.nvml = self._open_nvml()
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
            deadline = time.time() + 8.0       # nvidia-smi takes ~1 s to start sampling
            while not self.rows and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            r = [c.strip() for c in line.split(",")]
            try:
                reasons = {nm for k, nm in enumerate(self.NAMES) if len(r) > 5 + k and r[5 + k].lower() == "active"}
                self.rows.append((time.time(), float(r[1]), float(r[2]), reasons))
            except (ValueError, IndexError):
                pass

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()
        n = len(self.rows)
        deadline = time.time() + (0.5 if self.proc else 0.05)   # one more sample after the region
        while len(self.rows) == n and time.time() < deadline:
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        t0 = self.t0 if self.t0 is not None else self.rows[0][0]
        t1 = self.t1 if self.t1 is not None else self.rows[-1][0]
        slack = 0.15 if self.proc else 0.005
        rows = [r for r in self.rows if t0 <= r[0] <= t1 + slack]
        if not rows:            # region shorter than the sampling period: nearest sample
            rows = [min(self.rows, key=lambda r: abs(r[0] - 0.5 * (t0 + t1)))]
        reasons = set().union(*[r[3] for r in rows])
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# ----------------------------------------------------------- oracle (CPU) --
_ORACLE_SETUP = {}


def oracle_setup(w):
    """The oracle's grid and field window of workload w (built once per process:
    the field window of a full-size workload takes seconds on the host)."""
    import oracle as O
    from paper_2507_20719_b200 import inputs as I
    key = (w.name, tuple(w.ncell), w.slab_or_all())
    if key not in _ORACLE_SETUP:
        g = O.make_grid(w.ncell, w.length, w.bc, w.dt, w.c, w.planet_center, w.planet_radius)
        lo, EB = I.field_window(w.with_slab(0, w.ncell[0]) if w.slab_or_all() == (0, w.ncell[0]) else w, 2)
        _ORACLE_SETUP[key] = (g, O.FieldWindow(lo, EB.numpy()))
    return _ORACLE_SETUP[key]


def oracle_rate(w, parts_cpu, target_s, n_iter=3, all_cores=False):
    """Time the CPU oracle (mover + moments, one cycle) on a bounded sample of the
    workload's particles; returns (updates/s, sample description, cores).
    all_cores: the OpenMP build of the same source (mover over
    particle ranges per thread, per-thread node grids merged in thread order)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    g, F = oracle_setup(w)
    cores = O.omp_threads() if all_cores else 1
    mover = O.mover_par if all_cores else O.mover

    def moments(P, st):
        return O.moments_par(g, P, st) if all_cores else O.moments(g, P, st, with_abs=False)

    # the oracle deposits on the global grid; restrict the sample to this rank's
    # slab (rank 0) -- a global grid of the same shape is used for the timing
    def run(n_per_species):
        tot = 0
        t0 = time.perf_counter()
        for s, sp in enumerate(w.species):
            P = {k: parts_cpu[s][k][:n_per_species].numpy().copy() for k in "xyzuvwq"}
            st = np.zeros(len(P["x"]), dtype=np.int8)
            mover(g, F, sp.qom, n_iter, P, st, relativistic=w.relativistic)
            moments(P, st)
            tot += len(P["x"])
        return tot, time.perf_counter() - t0
    nmax = min(p["x"].numel() for p in parts_cpu)
    n0 = min(20000 * cores, nmax)
    tot, dt = run(n0)
    rate = tot / dt
    n1 = int(min(nmax, max(n0, rate * target_s / len(w.species))))
    tot, dt = run(n1)
    how = f"OpenMP build, {cores} threads" if all_cores else "single thread"
    return (tot / dt, f"{n1} particles per species (first {n1} in id order of rank 0's slab), 1 cycle, "
            f"mover+moments, {how}", cores)


def oracle_sample_parts(w, device="cpu"):
    from paper_2507_20719_b200 import inputs as I
    return I.make_species(w, device=device)


def run_reference(args):
    """Reference arm: the CPU oracle as it stands, timed on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    torch.set_num_threads(1)
    w, desc = workload(args, args.gpus, 0)
    # generate a bounded sub-slab of the workload on the CPU (same recipe)
    from paper_2507_20719_b200 import inputs as I
    sub = w.with_slab(0, max(1, min(w.slab_or_all()[1], 4)))
    parts = I.make_species(sub, device="cpu")
    vals = []
    for _ in range(args.warmup):
        oracle_rate(w, parts, min(2.0, args.cpu_seconds / 4), all_cores=True)
    for _ in range(args.steps):
        r, sample, cores = oracle_rate(w, parts, args.cpu_seconds / max(1, args.steps), all_cores=True)
        vals.append(r)
    v = statistics.median(vals)
    # one full step of the workload (all N GPUs' particles) at the sampled rate
    n_step = sum(I.species_upper_counts(w.with_slab(0, w.ncell[0])))
    line = {"impl": "reference", "metric": "particle updates/s (mover+moments)", "value": v,
            "unit": "particle updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": n_step / v * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "sample": sample,
                       "ms_per_step": f"projected: {n_step} particle updates at the sampled rate"},
            "cpu_baseline": {"value": v, "unit": "particle updates/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "particle updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def fp64_peak_tflops(seconds=1.5):
    """Sustained fp64 FMA throughput measured now on this GPU (tools/microbench/
    fp64peak.cu: back-to-back DFMA launches for `seconds`), or None."""
    import ctypes
    from paper_2507_20719_b200 import build_lib
    try:
        lib = ctypes.CDLL(build_lib.FP64PEAK_LIB)
        lib.fp64_fma_tflops.restype = ctypes.c_double
        lib.fp64_fma_tflops.argtypes = [ctypes.c_double]
        v = lib.fp64_fma_tflops(seconds * 1e3)
        return v if v > 0 else None
    except OSError:
        return None


def fp64_roofline(args, kname, n_alive, mover_ms_step, deposit_ms_step, rate_per_gpu, local):
    """%fp64 beside %HBM.  flops per update of each kernel:
    SASS-counted by ncu (2 DFMA + DADD + DMUL thread instructions + 512 per
    DMMA.8x8x4 warp instruction, per particle of the launch) in the committed
    capture profiles/fp64_ops.json (static: ncu cannot run inside the bench);
    peak: the sustained DFMA rate measured in this run, with its clocks."""
    path = os.path.join(ROOT, "profiles", "fp64_ops.json")
    if not os.path.exists(path) or args.relativistic or args.kernel == 1:
        return None
    ops = json.load(open(path))
    km = ops.get("kernels", {})
    mov = next((v for k, v in km.items() if k.startswith(kname)), None)
    dep = next((v for k, v in km.items() if k.startswith("deposit_tiled_kernel")), None)
    if mov is None or dep is None:
        return None
    with ClockSampler(local) as clk:
        clk.begin()
        peak = fp64_peak_tflops()
        clk.end()
    if not peak:
        return None
    f_mov, f_dep = mov["flops_per_update"], dep["flops_per_update"]
    achieved = n_alive * f_mov / (mover_ms_step / 1e3) / 1e12
    return {"bound": "alu", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "flops_per_update": f_mov,
            "deposit": {"flops_per_update": f_dep,
                        "achieved": n_alive * f_dep / (deposit_ms_step / 1e3) / 1e12 if deposit_ms_step else None},
            "step_frac": rate_per_gpu * (f_mov + f_dep) / (peak * 1e12),
            "peak_kind": "measured in this run: sustained DFMA, tools/microbench/fp64peak.cu",
            "peak_clocks": clk.summary(),
            "ops_source": {"kind": "static ncu capture (not this run)", "file": "profiles/fp64_ops.json",
                           "from": ops.get("source")}}


# --------------------------------------------------------------- GPU arm ----
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2507_20719_b200 import decomp, inputs as I, pic

    w, desc = workload(args, world, rank)
    nccl_id = decomp.broadcast_nccl_id(pic.pic_nccl_id) if world > 1 else None
    # the context runs on a stream of its own (CUDA-graph capture of whole
    # cycles needs one); torch work is ordered against it by synchronisation
    stream = torch.cuda.Stream()
    parts_cpu_sample = None
    want_sample = rank == 0 and world == 1 and not args.no_cpu_baseline
    if args.config in ("c3", "c4", "c5"):
        # full-size weak-scaling / magnetosphere slabs hold ~0.9-1.1 G particles
        # per GPU (the store alone is 136-165 GB): allocate it first (capacity =
        # particles before the planet cut, +2 % migration headroom with several
        # ranks) and draw the particles in host memory, sub-slab by sub-slab
        ub = I.species_upper_counts(w)
        cap = [int(n * (1.02 if world > 1 else 1.0)) + 65536 for n in ub]
        cfg = pic.make_config(w, rank=rank, nranks=world, capacity=cap, ghost=args.ghost,
                              transport=args.transport, kernel=args.kernel)
        need = pic.pic_workspace_bytes(cfg)
        free_b = torch.cuda.mem_get_info()[0]
        if need > free_b:
            raise SystemExit(f"{args.config}: store needs {need / 1e9:.1f} GB on rank {rank}, "
                             f"{free_b / 1e9:.1f} GB free: run it on more GPUs")
        ctx = pic.Context(cfg, nccl_id=nccl_id, stream=stream)
        # drawn on the device sub-slab by sub-slab and appended (pic_add_particles):
        # no host copy of the store, transient memory of one sub-slab
        for a, b, parts in I.iter_species_chunks(w, 64_000_000, device="cuda"):
            torch.cuda.synchronize()     # drawn on torch's stream, copied on libpic's
            for s, p in enumerate(parts):
                ctx.add_particles(s, p)
            if want_sample and parts_cpu_sample is None:
                parts_cpu_sample = [{k: v[:2_000_000].cpu() for k, v in p.items()} for p in parts]
            del parts
        ctx.sync()
    else:
        parts = I.make_species(w, device="cuda")
        torch.cuda.synchronize()         # drawn on torch's stream, copied on libpic's
        n_local = [p["x"].numel() for p in parts]
        face = w.ncell[1] * w.ncell[2]
        cap = [int(n * (1.35 if args.control else 1.08)) + 65536 + (4 * face * 64 if args.config == "c4s" else 0)
               for n in n_local]
        cfg = pic.make_config(w, rank=rank, nranks=world, capacity=cap, ghost=args.ghost,
                              transport=args.transport, kernel=args.kernel)
        ctx = pic.Context(cfg, nccl_id=nccl_id, stream=stream)
        for s, p in enumerate(parts):
            ctx.set_particles(s, p)
            if args.config == "c4s":
                # NEXT-3: wind injection at the x = 0 face with the bulk wind's parameters
                sp = w.species[s]
                ctx.set_injection(s, 64, sp.vth, sp.drift, float(p["q"][0].item()), 4242 + s)
        if want_sample:
            # bounded oracle sample: first particles of the store in id order (x-planes 0..)
            parts_cpu_sample = [{k: v[: min(v.numel(), 2_000_000)].cpu() for k, v in p.items()} for p in parts]
        del parts
    torch.cuda.empty_cache()
    lo, EB = I.field_window(w, args.ghost, device="cuda")
    torch.cuda.synchronize()
    ctx.set_fields(EB)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    barrier()    # every rank has its context, particles and fields before the first (collective) cycle
    for _ in range(args.warmup):
        ctx.cycle()
    ctx.sync()
    n_alive = sum(ctx.count(s) for s in range(len(w.species)))

    # ---- timed region (device time, CUDA events on the context stream).  With
    # --graph 1 the step is pic_cycle (replayed from CUDA graphs when libpic
    # allows it: peer transport or one rank, no injection), timed alone; the
    # per-phase kernel times (roofline, phase_ms) come from a second pass of the
    # same number of steps with CUDA events around every phase (pic_profile,
    # no graphs).  With --graph 0 one profiled pass gives both.
    def profiled_pass():
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        ctx.profile(True)
        barrier()
        torch.cuda.nvtx.range_push("bench_steps")   # ncu --nvtx --nvtx-include "bench_steps/"
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(args.steps):
            e0, e1, e2 = ev[k]
            e0.record(stream)
            ctx.mover(-1)
            e1.record(stream)
            ctx.moments(-1)
            ctx.exchange()
            e2.record(stream)
        end.record(stream)
        barrier()
        torch.cuda.nvtx.range_pop()
        prof = ctx.profile_read()
        ctx.profile(False)
        return start.elapsed_time(end), prof, ([a.elapsed_time(b) for a, b, c in ev], [b.elapsed_time(c) for a, b, c in ev])

    use_graph = bool(args.graph)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        if use_graph:
            ctx.set_graph(True)
            ctx.cycle()            # capture (or plain fallback), untimed
            ctx.cycle()
            barrier()
            clk.begin()
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            launches0 = ctx.launch_count()
            start.record(stream)
            for k in range(args.steps):
                ctx.cycle()
            end.record(stream)
            barrier()
            clk.end()
            t_ms = start.elapsed_time(end)
            launches = ctx.launch_count() - launches0
            ctx.set_graph(False)
            _, prof, (mover_ms, rest_ms) = profiled_pass()
        else:
            clk.begin()
            t_ms, prof, (mover_ms, rest_ms) = profiled_pass()
            clk.end()
            launches = ctx.launch_count() - launches0
    kps = {k: round(v[0] / args.steps, 4) for k, v in prof.items()}
    kps_ranks = [kps]
    if world > 1:
        kps_ranks = [None] * world
        dist.all_gather_object(kps_ranks, kps)
    stats = ctx.sync()
    tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    tot = torch.tensor([float(n_alive)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    t_ms = float(tt.item())
    total_updates = float(tot.item()) * args.steps
    value = total_updates / (t_ms / 1e3)

    # ---- roofline of the dominant kernel: the mover kernel (Eq. 2).  achieved =
    # its algorithmic bytes (read x, v: 48 B; write x, v: 48 B; plus the field
    # share 48 B per node / particles per cell) x particles / its event-timed
    # duration (pic_profile: CUDA events on the libpic stream around the mover
    # launches inside the timed region).  The whole step's fraction uses the
    # north_star figure 104 B + grid share.
    peak, peak_kind = measured_peaks()
    n_sp = len(w.species)
    ppc = w.species[0].ppc
    grid_share = (48.0 + 80.0 * n_sp) / (ppc * n_sp)
    b_mover = 96.0 + 48.0 / (ppc * n_sp)
    b_deposit = 56.0 + 80.0 / ppc
    mover_ms_step = prof["mover"][0] / args.steps
    deposit_ms_step = prof["deposit"][0] / args.steps
    mover_launch_ms = prof["mover"][0] / max(1, prof["mover"][1])
    achieved = n_alive * b_mover / (mover_ms_step / 1e3) / 1e9
    # traffic: NOT measured in this run (ncu cannot run inside the bench); the
    # DRAM bytes per update of the mover from the committed `ncu --set full`
    # capture named in `traffic_source`, attached only when that capture is of
    # this config and kernel family, scaled per launch (particles / species)
    traffic = None
    traffic_src = None
    ncu_pct = None
    kname = "mover_tiled_kernel" if args.kernel in (0, 2) else "mover_basic_kernel"
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == args.config and tj.get("kernel", "mover_tiled_kernel") == kname \
                    and not args.relativistic:
                # per launch: one mover launch moves every species sharing n_iter
                traffic = tj["mover_bytes_per_update"] * n_alive / max(1.0, prof["mover"][1] / args.steps)
                traffic_src = {"kind": "static ncu capture (not this run)", "file": "profiles/traffic.json",
                               "from": tj.get("source"), "bytes_per_update": tj["mover_bytes_per_update"]}
                ncu_pct = {k: tj[k] for k in ("mover_fp64_pipe_pct", "mover_issue_active_pct", "mover_dram_pct",
                                              "deposit_dram_pct") if k in tj}
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": kname,
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "ncu_utilisation_pct": ncu_pct,
            "bytes_per_update": b_mover, "launch_ms": mover_launch_ms,
            "launches_per_step": prof["mover"][1] / args.steps,
            "step_frac": (value / world) * (B_ALG_PARTICLE + grid_share) / (peak * 1e9),
            "step_bytes_per_update": B_ALG_PARTICLE + grid_share,
            "deposit": {"kernel": "deposit_tiled_kernel" if args.kernel in (0, 2) else "moments_basic_kernel",
                        "bytes_per_update": b_deposit, "ms_per_step": deposit_ms_step,
                        "achieved": n_alive * b_deposit / (deposit_ms_step / 1e3) / 1e9 if deposit_ms_step else None}}
    mover_avg = sum(mover_ms) / len(mover_ms)
    roof64 = fp64_roofline(args, kname, n_alive, mover_ms_step, deposit_ms_step, value / world, local)
    # the mover's binding unit: the shared-memory crossbar,
    # 128 B per SM cycle (B300_MICROARCH.md "LDS/STS"; a broadcast counts as
    # one access).  Wavefronts per update from the same static ncu capture as
    # `traffic`; the time is this run's, the peak at this run's median SM clock.
    roof_smem = None
    sm_mhz = clk.summary().get("sm_mhz")
    if traffic_src is not None and tj.get("mover_smem_wavefronts_per_update") and sm_mhz:
        wf = tj["mover_smem_wavefronts_per_update"]
        got = wf * 128 * n_alive / (mover_ms_step / 1e3) / 1e9
        n_sms = torch.cuda.get_device_properties(local).multi_processor_count
        top = 128 * n_sms * sm_mhz * 1e6 / 1e9
        roof_smem = {"bound": "smem", "kernel": kname, "achieved": got, "peak": top, "unit": "GB/s",
                     "frac": got / top, "wavefronts_per_update": wf,
                     "peak_kind": "128 B/cycle/SM x %d SMs x the median SM clock of this run (%.0f MHz)"
                                  % (n_sms, sm_mhz),
                     "wavefronts_source": {"kind": "static ncu capture (not this run)",
                                           "file": "profiles/traffic.json", "from": tj.get("source")}}

    # ---- e2e through the public API with host buffers (paper's discrete-GPU
    # cycle: fields host->device, moments device->host).  Every
    # step copies its field window in from pinned host memory and its moments
    # out to pinned host memory; the copies run on libpic's copy stream and
    # overlap the neighbouring steps' kernels (double-buffered fields, two
    # staging slots per species); the timed region ends after the last copy.
    e2e = None
    if not args.no_e2e:
        EB_h = EB.cpu().pin_memory()
        shape = ctx.moment_shape()
        mom_h = [torch.empty((10, shape[2], shape[1], shape[0]), dtype=torch.float64).pin_memory()
                 for _ in range(n_sp)]
        ctx.set_graph(use_graph)
        for _ in range(4):       # untimed: capture the graphs of both field buffers x store parities
            ctx.set_fields(EB_h)
            ctx.cycle()
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            ctx.set_fields(EB_h)
            ctx.cycle()
            for s in range(n_sp):
                ctx.get_moments_async(s, mom_h[s])
        ctx.join_copies()
        b.record(stream)
        barrier()
        te = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        n_alive2 = sum(ctx.count(s) for s in range(n_sp))
        tot2 = torch.tensor([float(n_alive2)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tot2, op=dist.ReduceOp.SUM)
        e2e = {"value": float(tot2.item()) * args.steps / (float(te.item()) / 1e3), "unit": "particle updates/s",
               "h2d_bytes_per_step": EB_h.numel() * 8,
               "d2h_bytes_per_step": sum(m.numel() * 8 for m in mom_h)}
        ctx.sync()

    # ---- NEXT-2: the field solver's sources (Eq. 5-6) from this step's moments
    next2 = None
    if world == 1:
        ctx.implicit_sources()                      # warm-up (allocates the outputs)
        nx_, ny_, nz_ = ctx.moment_shape()
        a2 = torch.cuda.Event(enable_timing=True)
        b2 = torch.cuda.Event(enable_timing=True)
        reps = 5
        a2.record(stream)
        for _ in range(reps):
            ctx.implicit_sources()
        b2.record(stream)
        torch.cuda.synchronize()
        ms2 = a2.elapsed_time(b2) / reps
        nodes = nx_ * ny_ * nz_
        # algorithmic bytes per node: 10 moments x S in, B in, chi 9 + J-hat 3 +
        # rho-hat 1 out, J-hat read back for the divergence
        b_node = 80 * n_sp + 24 + 104 + 24
        next2 = {"what": "chi, rho-hat, J-hat (Eq. 5-6) over the owned nodes, incl. output allocation and sync",
                 "ms_per_call": ms2, "nodes": nodes, "bytes_per_node": b_node,
                 "achieved_gbs": nodes * b_node / (ms2 / 1e3) / 1e9}

    # ---- NEXT-3 particle control: one split pass (+20 % target) and one
    # coalescence pass (back to the initial count), timed on the device
    next3 = None
    if args.control and world == 1:
        res = {}
        for name, fac in (("split", 1.2), ("coalesce", 0.9)):
            n0 = [ctx.count(s) for s in range(n_sp)]
            a3 = torch.cuda.Event(enable_timing=True)
            b3 = torch.cuda.Event(enable_timing=True)
            a3.record(stream)
            acts = [ctx.control(s, int(fac * n0[s]) if name == "split" else int(n_alive / n_sp * fac), 0.05, 0.1,
                                w.species[s].vth / 2, 7) for s in range(n_sp)]
            b3.record(stream)
            torch.cuda.synchronize()
            n1 = [ctx.count(s) for s in range(n_sp)]
            res[name] = {"ms": a3.elapsed_time(b3), "actions": acts, "particles_before": sum(n0),
                         "particles_after": sum(n1)}
        next3 = {"what": "pic_control on every species (count sync, pass, order rebuild)", **res}

    # ---- NEXT-4: velocity histogram + Gaussian-mixture fit per species
    next4 = None
    if args.gmm and world == 1:
        import time as _t
        res = []
        for s in range(n_sp):
            vmax = 5.0 * w.species[s].vth
            t0 = _t.perf_counter()
            a, mu, sg, h, clipped = ctx.gmm(s, 24, vmax, 4, 50)
            res.append({"species": w.species[s].name, "ms": (_t.perf_counter() - t0) * 1e3, "bins": 24, "M": 4,
                        "n_em": 50, "alpha": a.tolist(), "clipped": clipped})
        next4 = {"what": "pic_gmm per species: 24^3 velocity bins, 4 components, 50 EM iterations (host-timed, synchronous)",
                 "fits": res}

    cpu = cpu1 = None
    if parts_cpu_sample is not None:
        threads = torch.get_num_threads()
        torch.set_num_threads(1)
        r1, sample1, _ = oracle_rate(w, parts_cpu_sample, args.cpu_seconds / 2)
        ra, samplea, cores = oracle_rate(w, parts_cpu_sample, args.cpu_seconds / 2, all_cores=True)
        torch.set_num_threads(threads)
        cpu = {"value": ra, "unit": "particle updates/s", "cores": cores, "kind": "oracle", "sample": samplea,
               "single_thread": {"value": r1, "unit": "particle updates/s", "cores": 1, "kind": "oracle",
                                 "sample": sample1}}
        cpu1 = dict(cpu["single_thread"])

    if rank == 0:
        line = {
            "metric": "particle updates/s (mover+moments)", "value": value, "unit": "particle updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "particles_per_gpu": n_alive, "cells_per_gpu": [w.slab_or_all()[1] - w.slab_or_all()[0]] + list(w.ncell[1:]),
                       "kernel": ["auto", "basic", "tiled"][args.kernel], "transport": (["nccl", "peer"][int(ctx.peer)] if world > 1 else None),
                       "l2": "inputs (%.2f GB per GPU) exceed the 126 MB L2; no flush" % (n_alive * 64 / 1e9),
                       "parallelism": f"x-slabs{world}",
                       "step": ("pic_cycle, replayed from CUDA graphs where libpic allows (pic_set_graph); kernel "
                                "times from a second, profiled pass" if use_graph else
                                "pic_mover + pic_moments + pic_exchange, plain launches, profiled")},
            "roofline": roof,
            "roofline_fp64": roof64,
            "roofline_smem": roof_smem,
            "parity_report": "profiles/r02_parity_report.json (tools/parity_report.py: max error / bound per "
                             "config clone, kernel family and species; not run by the bench)",
            "cpu_baseline": cpu,                  # the oracle on every host core (OpenMP build)
            "cpu_baseline_1core": cpu1,           # the single-threaded parity checker
            "e2e": e2e,
            "next2_sources": next2,
            "next3_control": next3,
            "next4_gmm": next4,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "phase_ms": {"mover+order": mover_avg, "moments+exchange": sum(rest_ms) / len(rest_ms),
                         "kernels_per_step": kps,
                         **({"kernels_per_step_ranks": kps_ranks} if world > 1 else {})},
            "stats": stats,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
