#!/usr/bin/env python
"""Host-side transfer probe for the host-buffer decode API:
pinned H2D / D2H / both directions at once, pageable->pinned host copies, and
the cost of fresh vs cached output allocations.  Informs the pipeline design,
not a product number."""
import json
import os
import time

import numpy as np
import torch


def ev_time(fn, reps=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def wall(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def main():
    nb = 600 * 2**20
    out = {"cores": len(os.sched_getaffinity(0)), "torch_threads": torch.get_num_threads()}
    hp = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    hp2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    out["h2d_pinned_GBs"] = nb / ev_time(lambda: d.copy_(hp, non_blocking=True)) / 1e9
    out["d2h_pinned_GBs"] = nb / ev_time(lambda: hp.copy_(d, non_blocking=True)) / 1e9
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(hp, non_blocking=True)
        with torch.cuda.stream(s2):
            hp2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    out["bidir_total_GBs"] = 2 * nb / ev_time(both) / 1e9
    pg = np.ones(nb, dtype=np.uint8)
    out["h2d_pageable_GBs"] = nb / wall(lambda: (d.copy_(torch.from_numpy(pg)), torch.cuda.synchronize())) / 1e9
    out["pageable_to_pinned_torch_GBs"] = nb / wall(lambda: hp.copy_(torch.from_numpy(pg))) / 1e9
    out["np_copyto_GBs"] = nb / wall(lambda: np.copyto(hp.numpy(), pg)) / 1e9
    out["np_empty_touch_s"] = wall(lambda: np.empty(nb, dtype=np.uint8).fill(0))
    out["np_empty_s"] = wall(lambda: np.empty(nb, dtype=np.uint8))
    t0 = time.perf_counter()
    x = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    out["pinned_alloc_first_s"] = time.perf_counter() - t0
    del x
    t0 = time.perf_counter()
    x = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    out["pinned_alloc_cached_s"] = time.perf_counter() - t0
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
