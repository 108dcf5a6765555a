#!/usr/bin/env python
"""Turn an ncu --csv launch list (dram__bytes_read/write.sum, gpu__time_duration.sum)
into profiles/<round>/ncu_traffic.json records bench.py reads for roofline.traffic.

  python tools/ncu_traffic.py gpurun_out/traffic.csv --tag cnu_phi --gamma 4096 --match "cnu_kernel<24, 2, 1, 2" --out profiles/r01/ncu_traffic.json
"""
import argparse
import csv
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--gamma", type=int, required=True)
    ap.add_argument("--match", required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr, launches = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if a.match not in d["Kernel Name"]:
                continue
            unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
            v = float(d["Metric Value"].replace(",", "")) * unit.get(d["Metric Unit"], 1)
            launches.setdefault(d["ID"], {})[d["Metric Name"]] = v
    recs = [v for v in launches.values() if "dram__bytes_read.sum" in v]
    rd = sum(v["dram__bytes_read.sum"] for v in recs) / len(recs)
    wr = sum(v["dram__bytes_write.sum"] for v in recs) / len(recs)
    ns = sum(v.get("gpu__time_duration.sum", 0) for v in recs) / len(recs)
    out = json.load(open(a.out)) if os.path.exists(a.out) else []
    out = [o for o in out if not (o["tag"] == a.tag and o["gamma"] == a.gamma)]
    out.append({"tag": a.tag, "gamma": a.gamma, "kernel": a.match, "launches": len(recs),
                "dram_read": int(rd), "dram_write": int(wr), "dram_bytes": int(rd + wr),
                "ncu_duration_ns": int(ns), "source": os.path.basename(a.csv)})
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out[-1]))


if __name__ == "__main__":
    main()
