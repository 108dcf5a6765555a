"""GPU: the sharded Monte-Carlo driver with 2 ranks sharing the one GPU (gloo
carries the counter all_reduce here; NCCL in production needs one GPU per
rank).  Totals must equal the single-process campaign and the reference."""
import json
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1204_0334_b200 as q
    lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    cfg = q.SimulationConfig(code_id="toy", ebn0_db=[2.0, 3.0], iterations=8, processors=2, gamma=8,
                             stop_block_errors=15, max_frames=2000, seed=5)
    res = q.run_block_simulation(lay, cfg, gamma_kernel=32)
    code = q.unwrap_qc(q.multiplicative_shifts(2, 4, 8))
    cfg2 = q.SimulationConfig(code_id="toy", ebn0_db=[2.0], iterations=8, processors=2, gamma=8,
                              stop_block_errors=10, max_frames=500, seed=5, stream_segment_frames=6)
    res2 = q.run_stream_simulation(code, cfg2, gamma_kernel=32)
    # early-stop campaign through lane recycling, batches round-robin over ranks
    lay3 = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(4, 24, 29)))
    cfg3 = q.SimulationConfig(code_id="es", ebn0_db=[2.6], iterations=20, gamma=32, stop_block_errors=9,
                              max_frames=4000, seed=2, early_stop=True)
    res3 = q.run_block_simulation(lay3, cfg3, gamma_kernel=256)
    out[rank] = ([r.row()[:10] for r in res], [r.row()[:10] for r in res2], [r.row()[:8] for r in res3])
    dist.destroy_process_group()


def test_two_ranks_share_counters():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    camp = json.load(open(os.path.join(GOLDEN, "campaigns.json")))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(2, _port(), out), nprocs=2, join=True)
    assert out[0] == out[1]
    assert out[0][0] == camp["toy_block"]
    assert out[0][1] == camp["toy_stream"]
    from oracle import campaign, qc as oqc
    want = campaign.block_point(oqc.qc_layout(oqc.array_code_shifts(4, 24, 29), 29), 2.6, 0, iters=20,
                                gamma=32, seed=2, stop=9, max_frames=4000, early_stop=True)
    assert tuple(out[0][2][0][5:8]) == want
