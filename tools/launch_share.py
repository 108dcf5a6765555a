#!/usr/bin/env python
"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum
--csv launch list (cold-cache, serialised: compare shares, not absolutes)."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
            scale = {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(d["Metric Unit"], 1)
            tot[name] += float(d["Metric Value"].replace(",", "")) * scale
            cnt[name] += 1
    all_ns = sum(tot.values())
    print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / all_ns:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1])
