#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): device
time per kernel and its share of the listed launches (cold-cache, serialised:
compare shares, not absolutes).   python tools/launch_summary.py list.csv"""
import collections
import csv
import json
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui, mi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
    tot, n = collections.Counter(), collections.Counter()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0].replace("void ", "")
        k = k.split("<")[0] if "CUB_" in k else k
        tot[k] += float(r[vi].replace(",", "")) * scale[r[ui]]
        n[k] += 1
    T = sum(tot.values())
    out = {k: {"ms": round(v, 4), "share": round(v / T, 4), "launches": n[k]} for k, v in tot.most_common()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
