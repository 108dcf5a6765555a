"""CPU, world_size 2 over gloo: the multi-GPU campaign's sharding + counter reduce.

Each rank computes the per-batch counts of its own batches with the oracle
(the GPU path does the same with the kernels), writes them into its slice of
the round's counter array, all_reduce(SUM) merges them, and both ranks apply
the ordered stop rule -- the totals must equal a single-process run.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import campaign, qc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1204_0334_b200.dist import ordered_prefix, sum_counts
    lay = qc.qc_layout(qc.array_code_shifts(2, 4, 8), 8)
    from oracle import channel
    sigma = channel.ebn0_to_sigma(2.0, 0.5)
    campaign._init(lay=lay, seed=5, sigma=sigma, gamma=8, iters=8, lane0=0)
    units, tot, done, rnd = 2, (0, 0, 0), False, 0
    while not done:
        allc = torch.zeros((world * units, 3), dtype=torch.int64)
        for u in range(units):
            b = (rnd * world + rank) * units + u
            allc[rank * units + u] = torch.tensor(campaign.block_task(b))
        sum_counts(allc, dist.group.WORLD)
        tot, done, _ = ordered_prefix(allc.numpy(), 15, 2000, tot)
        rnd += 1
    out[rank] = tot
    dist.destroy_process_group()


def test_two_rank_counts_equal_single_process():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    lay = qc.qc_layout(qc.array_code_shifts(2, 4, 8), 8)
    single = campaign.block_point(lay, 2.0, 0, iters=8, gamma=8, seed=5, stop=15, max_frames=2000)
    assert out[0] == out[1] == single
