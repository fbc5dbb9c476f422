#!/usr/bin/env python3
"""Summarise an ncu report of the fused kernel into profiles/ (markdown + json).

    python tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep profiles/TAG --particles N

Reads the raw page (key counters) and the source page (per-line instructions
and stall samples) with `ncu -i`; no GPU needed.  The json carries the DRAM
traffic per launch and per particle update that bench.py reports as
roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__inst_executed_pipe_fp64.sum", "smsp__warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
]


LAUNCH = 0


def ncu_csv(rep, *args):
    out = subprocess.check_output(["ncu", "-i", rep, "--csv", "--launch-skip", str(LAUNCH), "--launch-count", "1"]
                                  + list(args), stderr=subprocess.DEVNULL).decode()
    return list(csv.reader(io.StringIO(out)))


def fp64_flops(m):
    """SASS-counted fp64 flops: 2 per DFMA, 1 per DADD / DMUL thread instruction,
    512 per DMMA.8x8x4 warp instruction (8 x 8 x 4 FMAs)."""
    g = lambda k: m.get(k, (0.0, ""))[0]
    return (2 * g("sm__sass_thread_inst_executed_op_dfma_pred_on.sum") + g("sm__sass_thread_inst_executed_op_dadd_pred_on.sum")
            + g("sm__sass_thread_inst_executed_op_dmul_pred_on.sum") + 512 * g("sm__inst_executed_pipe_tensor_subpipe_dmma.sum"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out_prefix")
    ap.add_argument("--particles", type=float, required=True, help="particles processed by the profiled launch")
    ap.add_argument("--title", default="")
    ap.add_argument("--launch", type=int, default=0, help="index of the profiled launch in the report")
    a = ap.parse_args()
    global LAUNCH
    LAUNCH = a.launch
    rows = ncu_csv(a.rep, "--page", "raw")
    h, units, vals = rows[0], rows[1], rows[2]
    kname = vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    m = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            try:
                m[k] = (float(vals[i].replace(",", "")), units[i])
            except ValueError:
                pass

    def val(k, unit_scale):
        v, u = m[k]
        return v * unit_scale.get(u, 1.0)
    t_ms = val("gpu__time_duration.sum", {"ms": 1, "msecond": 1, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3})
    gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
    rd = val("dram__bytes_read.sum", gb)
    wr = val("dram__bytes_write.sum", gb)
    # source page
    src = ncu_csv(a.rep, "--page", "source", "--print-source", "cuda,sass")
    cur, hdr, lines = None, None, []
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 8 and r[0].isdigit():
            try:
                ie = int(r[hdr.index("Instructions Executed")])
                st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except (ValueError, IndexError):
                continue
            stalls = {k[6:]: int(r[i]) for i, k in enumerate(hdr)
                      if k.startswith("stall_") and "Not Issued" not in k and r[i].isdigit()}
            lines.append((cur, int(r[0]), r[1].strip()[:90], ie, st, stalls))
    tot_i = sum(x[3] for x in lines) or 1
    tot_s = sum(x[4] for x in lines) or 1
    reasons = collections.Counter()
    for x in lines:
        reasons.update(x[5])
    rs = sum(reasons.values()) or 1
    summary = {
        "kernel": kname, "title": a.title, "launch_ms": t_ms, "particles": a.particles,
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
        "traffic_bytes_per_update": (rd + wr) / a.particles,
        "dram_gbs": (rd + wr) / (t_ms * 1e-3) / 1e9,
        "metrics": {k: v for k, (v, u) in m.items()},
        "warp_instr_per_particle": tot_i / a.particles,
        "fp64_flops_per_particle": fp64_flops(m) / a.particles,
        "stall_reasons_pct": {k: round(100.0 * v / rs, 1) for k, v in reasons.most_common(10)},
    }
    with open(a.out_prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(a.out_prefix + ".md", "w") as f:
        f.write(f"# ncu summary: {a.title or kname}\n\n`{kname}`\n\n")
        f.write(f"- launch time (ncu, clock-control none): {t_ms:.3f} ms for {a.particles:.4g} particles\n")
        f.write(f"- DRAM read {rd/1e9:.3f} GB + write {wr/1e9:.3f} GB = {(rd+wr)/a.particles:.1f} B per particle update "
                f"({(rd+wr)/(t_ms*1e-3)/1e9:.0f} GB/s)\n")
        for k, (v, u) in m.items():
            f.write(f"- `{k}` = {v:g} {u}\n")
        f.write(f"\nWarp instructions per particle: {tot_i / a.particles:.1f}; "
                f"fp64 flops per particle (SASS-counted): {fp64_flops(m) / a.particles:.1f}\n\n")
        f.write("Stall reasons (share of samples): " +
                ", ".join(f"{k} {100.0*v/rs:.1f}%" for k, v in reasons.most_common(8)) + "\n\n")
        f.write("| file:line | warp instr / particle | stall % | top stall | source |\n|---|---|---|---|---|\n")
        for x in sorted(lines, key=lambda t: -t[4])[:30]:
            top = max(x[5].items(), key=lambda kv: kv[1])[0] if x[5] else ""
            f.write(f"| {x[0]}:{x[1]} | {x[3]/a.particles:.2f} | {100.0*x[4]/tot_s:.1f} | {top} | `{x[2].replace('|','/')}` |\n")
    print(json.dumps({k: summary[k] for k in ("kernel", "launch_ms", "traffic_bytes_per_update", "dram_gbs",
                                               "warp_instr_per_particle", "fp64_flops_per_particle")}))


if __name__ == "__main__":
    main()
