#!/usr/bin/env python
"""Rough L2 vs HBM read bandwidth on this GPU: repeated reductions over buffers
that fit in L2 (8-64 MB) and one that does not (2 GB).  Informs design choices
(DESIGN.md), not a product number."""
import json

import torch


def bw(mb, reps=50):
    x = torch.ones(int(mb * 2**20 // 4), dtype=torch.float32, device="cuda")
    for _ in range(3):
        x.sum()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        x.sum()
    b.record()
    torch.cuda.synchronize()
    return x.numel() * 4 * reps / (a.elapsed_time(b) / 1e3) / 1e9


if __name__ == "__main__":
    print(json.dumps({f"{mb}MB_read_GBs": round(bw(mb), 1) for mb in (8, 16, 32, 48, 64, 96, 2048)}))
