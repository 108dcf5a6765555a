#!/usr/bin/env python
"""Summarise ncu --set full reports (.ncu-rep) as markdown: duration, DRAM
bytes vs algorithmic, throughput, occupancy, issue activity, top stall reasons.

  python tools/ncu_summary.py gpurun_out/prof_cnu.ncu-rep [--alg-bytes N] ...
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]


def summarize(path, alg=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"### {path.split('/')[-1]}", "", "| metric | value |", "|---|---|"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        for k, label in KEYS:
            if k in d:
                lines.append(f"| {label} | {d[k]} {u.get(k, '')} |")
        if alg:
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            f = scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
            lines.append(f"| DRAM traffic / algorithmic bytes | {(rd + wr) * f / alg:.3f} |")
        stalls = {k: float(v.replace(",", "") or 0) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        lines.append("| top stalls (warps per issue) | " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for k, v in top) + " |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    alg = None
    if "--alg-bytes" in args:
        i = args.index("--alg-bytes")
        alg = float(args[i + 1])
        del args[i:i + 2]
    for p in args:
        print(summarize(p, alg))
