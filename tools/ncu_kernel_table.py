#!/usr/bin/env python
"""Per-kernel DRAM throughput table from an ncu --csv launch list with
dram__bytes_read.sum, dram__bytes_write.sum and gpu__time_duration.sum:
mean duration, mean DRAM bytes, achieved GB/s and fraction of the measured
HBM peak (MEASURED_PEAKS.json) for every kernel name.  ncu replays are
cold-cache and serialised, so these are per-kernel DRAM rates, not step times.

  python tools/ncu_kernel_table.py gpurun_out/all_kernels.csv > profiles/r01/ncu_every_kernel.md
"""
import collections
import csv
import json
import os
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
        "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}


def main(path):
    peak = 6554.6
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peak = float(json.load(open(mp))["hbm_gbs"])
    rows = list(csv.reader(open(path)))
    hdr, launches = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
            name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
            launches.setdefault(d["ID"], {"name": name})[d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for L in launches.values():
        if "gpu__time_duration.sum" not in L:
            continue
        a = agg[L["name"]]
        a[0] += 1
        a[1] += L["gpu__time_duration.sum"]
        a[2] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    print(f"DRAM throughput per kernel (ncu, cold-cache serialised replays), peak = {peak} GB/s "
          f"(MEASURED_PEAKS.json copy)\n")
    print("| kernel | launches | mean us | mean DRAM MB | DRAM GB/s | of peak |\n|---|---|---|---|---|---|")
    for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t / 1e9 if t else 0.0
        print(f"| `{name}` | {n} | {t / n * 1e6:.1f} | {b / n / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1])
