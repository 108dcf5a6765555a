#!/usr/bin/env python
"""HBM bandwidth at different read/write mixes (torch elementwise kernels over
1-2 GB operands): read-only reduction, copy (1:1), add (2:1), addcmul (3:1).
Calibrates the roofline denominator for kernels whose traffic is read-heavy
(the compact decode moves ~73% reads), next to MEASURED_PEAKS.json's copy."""
import json

import torch


def ev(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    n = 1 << 28                      # 1 GiB of fp32 per operand
    x, y, z, o = (torch.rand(n, device="cuda") for _ in range(4))
    out = {}
    s = torch.empty((), device="cuda")
    out["read_only_GBs"] = 4 * n / ev(lambda: torch.sum(x, dim=0, out=s)) / 1e9
    out["copy_1to1_GBs"] = 8 * n / ev(lambda: o.copy_(x)) / 1e9
    out["add_2to1_GBs"] = 12 * n / ev(lambda: torch.add(x, y, out=o)) / 1e9
    out["addcmul_3to1_GBs"] = 16 * n / ev(lambda: torch.addcmul(x, y, z, out=o)) / 1e9
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
