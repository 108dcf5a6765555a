"""GPU: the sharded Monte-Carlo driver with 2 ranks sharing the one GPU (gloo
carries the counter all_reduce here; NCCL in production needs one GPU per
rank).  Totals must equal the single-process campaign and the reference."""
import json
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp
from conftest import GOLDEN, REPO

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
    mgr = mp.get_context("spawn").Manager()     # never fork after CUDA init
    out = mgr.dict()
    mp.spawn(_rank, args=(2, _port(), out), nprocs=2, join=True)
    assert out[0] == out[1]
    assert out[0][0] == camp["toy_block"]
    assert out[0][1] == camp["toy_stream"]
    from oracle import campaign, qc as oqc
    want = campaign.block_point(oqc.qc_layout(oqc.array_code_shifts(4, 24, 29), 29), 2.6, 0, iters=20,
                                gamma=32, seed=2, stop=9, max_frames=4000, early_stop=True)
    assert tuple(out[0][2][0][5:8]) == want


def _bench(args, env_extra=None):
    import subprocess
    import sys
    repo = REPO
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), *args], capture_output=True, text=True,
                       env=env, timeout=900, cwd=repo)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line), r.stderr


def test_bench_gpus_2_entry_path_matches_one_rank():
    """`python bench.py --gpus 2` (no torchrun env) launches 2 ranks itself; with
    gloo both share the one GPU.  Rank r of step s decodes lanes (s*W + r)*gamma,
    so 2 ranks x 256 lanes cover the lanes of 1 rank x 512: the summed counters
    of the last step must be identical."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    common = ["--steps", "3", "--warmup", "3", "--no-e2e", "--stream-gamma", "0", "--no-cpu",
              "--sustain-s", "0"]
    two, err = _bench(["--gpus", "2", "--gamma", "256", *common], {"QCB_DIST_BACKEND": "gloo"})
    one, _ = _bench(["--gpus", "1", "--gamma", "512", *common])
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["communicator"]["world_size"] == 2 and two["communicator"]["ranks_summed"] == 2
    assert "launching 2 ranks" in err
    assert two["counts_last_step"] == one["counts_last_step"]
    assert two["counts_last_step"]["frames"] == 512
